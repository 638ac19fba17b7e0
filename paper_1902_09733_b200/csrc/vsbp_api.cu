// vsbp_api.cu -- the C ABI (include/vsbp.h): context, parameter quantisation,
// workspace plan and the launch sequence of hierarchical BP (SURVEY §3 call
// stacks).  Host code only; every device step is a kernel in bp_kernels.cu or
// pipeline_kernels.cu.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>

#include "vsbp.h"
#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

constexpr int EV_RING = 1024;  // pending level timings (bp_timing_enable)

struct vsbp_bp {
    int W, H, L, levels, iters;
    int lam_q, tau_d, tau_q, S;
    int Lp, nch, G, log2G;
    int msg_bytes_opt, msg_bytes, kernel;
    int dimg;  // level-0 data term computed from the images inside the update (no D_0 traffic)
    int final_fuse;  // VSBP_OPT_FINAL: last level-0 iteration fused with the WTA (messages not stored)
    int final_ran;   // the last call fused it: level-0 messages of the last colour are stale
    int pair_fuse;   // VSBP_OPT_PAIR: two checkerboard iterations per launch (k_update_pair)
    int pair_band;   // rows per CTA band of k_update_pair
    long long pair_min_px;  // VSBP_OPT_PAIR = 1: fuse levels of at least this many pixels
    int mcur[16];    // which of the level's two message arrays holds its current messages
    int Wl[16], Hl[16], Wcl[16];
    int dbytes[16];
    // workspace plan (bytes) for ws_batch pairs
    size_t d_off[16], m_off[16], m2_off[16], total;  // m2_off: the second message array (0: none)
    void *ws;
    size_t ws_bytes;
    int ws_batch;
    int last_B;
    const uint8_t *last_left, *last_right;  // the last call's images (debug cost export)
    // live timing of the a4 launches (bp_timing_enable)
    // a FIFO ring of EV_RING (start, end) event pairs, one per level per call,
    // drained without blocking as the events complete
    int timing;
    int ev_head, n_pending;
    cudaEvent_t ev[EV_RING][2];
    int ev_level[EV_RING];
    int ev_launches[EV_RING];
    double ev_bytes[EV_RING];
    double acc_ms[16], acc_bytes[16];
    int64_t acc_launches[16];
};

namespace {

thread_local char g_errbuf[256];
thread_local uint64_t g_launches;

int cuda_fail(cudaError_t e)
{
    snprintf(g_errbuf, sizeof g_errbuf, "CUDA error: %s", cudaGetErrorString(e));
    return VSBP_ECUDA;
}

#define CK(expr)                                  \
    do {                                          \
        cudaError_t e_ = (expr);                  \
        if (e_ != cudaSuccess) return cuda_fail(e_); \
    } while (0)

long long rha(double v) { return v >= 0 ? (long long)std::floor(v + 0.5) : -(long long)std::floor(-v + 0.5); }

int bytes_for_max(long long vmax)
{
    if (vmax <= 255) return 1;
    if (vmax <= 65535) return 2;
    return 4;
}

size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

bool use_pair(const vsbp_bp *c, int l, int B);
int pair_band_of(const vsbp_bp *c, int l);

void plan(vsbp_bp *c, int batch)
{
    size_t off = 0;
    for (int l = 0; l < c->levels; ++l) {
        c->d_off[l] = off;
        off = align256(off + (size_t)batch * 2 * c->Hl[l] * c->Wcl[l] * c->Lp * c->dbytes[l]);
    }
    for (int l = 0; l < c->levels; ++l) {
        c->m_off[l] = off;
        off = align256(off + (size_t)batch * 8 * c->Hl[l] * c->Wcl[l] * c->Lp * c->msg_bytes);
    }
    for (int l = 0; l < c->levels; ++l) {
        c->m2_off[l] = 0;
        if (use_pair(c, l, batch)) {  // monotone in B: a call with B <= batch never needs more
            c->m2_off[l] = off;
            off = align256(off + (size_t)batch * 8 * c->Hl[l] * c->Wcl[l] * c->Lp * c->msg_bytes);
        }
    }
    c->total = off;
}

// the level's current message array (k_update_pair ping-pongs between two)
inline char *msg_base(const vsbp_bp *c, char *ws, int l)
{
    return ws + (c->mcur[l] ? c->m2_off[l] : c->m_off[l]);
}

vsbp::Geom geom(const vsbp_bp *c, int B, int l)
{
    vsbp::Geom g;
    g.B = B;
    g.W = c->Wl[l];
    g.H = c->Hl[l];
    g.Wc = c->Wcl[l];
    const int lp = l + 1 < c->levels ? l + 1 : l;
    g.Wp = c->Wl[lp];
    g.Hp = c->Hl[lp];
    g.Wcp = c->Wcl[lp];
    g.L = c->L;
    g.Lp = c->Lp;
    g.nch = c->nch;
    g.G = c->G;
    g.log2G = c->log2G;
    return g;
}

inline char *wsp(const vsbp_bp *c) { return (char *)c->ws; }

// The packed kernel (bp_fast.cu) is exact when messages are u8 (tau_q <= 255 <= 2S,
// so the 3-tap stencil is the truncated-linear envelope), the level's costs are
// u8/u16 and every belief fits 16 bits, and L <= 512 (9-bit WTA key).
bool use_fast(const vsbp_bp *c, int l)
{
    if (c->kernel != 0 || c->msg_bytes != 1 || c->S != 128 || c->tau_q > 255 || c->L > 512) return false;
    if (c->dbytes[l] > 2) return false;
    if ((long long)8 * c->Hl[l] * c->Wcl[l] * c->Lp >= (1ll << 31)) return false;  // 32-bit offsets per pair
    const long long dmax = ((long long)c->lam_q * c->tau_d) << (2 * l);
    return dmax + 4LL * c->tau_q < 65536LL;
}

// level 0 of the packed kernel computes its data term from the grey images
bool use_dimg(const vsbp_bp *c) { return c->dimg && use_fast(c, 0) && c->dbytes[0] == 1 && c->tau_d <= 255; }
// VSBP_OPT_DIMG = 2: only the one-iteration level-0 launches compute the data term from
// the images; D_0 is still stored for the two-iteration kernel
bool dimg_only_singles(const vsbp_bp *c) { return use_dimg(c) && c->dimg == 2; }
// k_final_fast: packed level-0 update with u8 costs read from memory, a normal
// (MODE 0) last iteration, and a left neighbour for every colour-A pixel but x = 0
bool use_final(const vsbp_bp *c)
{
    return c->final_fuse && use_fast(c, 0) && !use_dimg(c) && c->dbytes[0] == 1 && c->iters >= 2 && c->W >= 2 &&
           (c->final_fuse != 3 || c->G <= 32);
}

// two iterations per launch (k_update_pair): the packed kernel with D from memory,
// at least three iterations (the last one of every level stays a single launch: its
// messages must all be stored -- the WTA, the up-copy and the exports read both
// colours), and one Lp chunk per lane group that fits the CTA
bool use_pair(const vsbp_bp *c, int l, int B)
{
    if (!c->pair_fuse || !use_fast(c, l) || c->iters < 3 || c->G > 32) return false;
    if (l == 0 && use_dimg(c) && !dimg_only_singles(c)) return false;
    if (c->pair_fuse == 2) return true;  // every level (tests)
    // a CTA walks its band row by row, so small levels have too few CTAs to fill the
    // GPU (levels 2-4 of C2 measured 1.8-2.3x slower fused)
    const long long px = (long long)c->Wl[l] * c->Hl[l];
    if (c->dbytes[l] == 1) return px >= c->pair_min_px;
    if (c->pair_fuse == 3) return false;  // u8-cost levels only
    // 1 (default): u16-cost levels too, when the call holds >= 2M of their pixels and
    // each pair >= 10K (C5 level 1 fused 8466 -> 8586 pairs/s, level 2 with
    // 16-row bands 8611 -> 8638; C4 level 1 0.191 -> 0.183 ms per pair; C4 level 2
    // (64K px x 8 pairs) 0.052 -> 0.066 ms)
#ifndef VSBP_U16_MIN_PX
#define VSBP_U16_MIN_PX 10000
#endif
#ifndef VSBP_U16_MIN_BATCH_PX
#define VSBP_U16_MIN_BATCH_PX 2000000
#endif
    return px >= VSBP_U16_MIN_PX && px * B >= VSBP_U16_MIN_BATCH_PX;
}

// rows per CTA band of k_update_pair on level l: pair_band, and 16 on levels shorter
// than two bands (4x the CTAs for the serial row walk: C5 level 2 fused gained only so)
int pair_band_of(const vsbp_bp *c, int l) { return c->Hl[l] < 2 * c->pair_band ? 16 : c->pair_band; }

// beliefs of level l fit 15 bits: the signed one-instruction normalise applies
bool fast_signed(const vsbp_bp *c, int l)
{
    const long long dmax = ((long long)c->lam_q * c->tau_d) << (2 * l);
    return dmax + 4LL * c->tau_q < 32768LL;
}

vsbp::FastArgs fast_args(const vsbp_bp *c, int l, char *ws, int32_t *disp)
{
    vsbp::FastArgs a;
    const int lp = l + 1 < c->levels ? l + 1 : l;
    a.M = (uint8_t *)msg_base(c, ws, l);
    a.Mw = c->m2_off[l] ? (uint8_t *)(ws + (c->mcur[l] ? c->m_off[l] : c->m2_off[l])) : nullptr;
    a.Mp = (const uint8_t *)msg_base(c, ws, lp);
    a.disp = disp;
    a.W = c->Wl[l];
    a.H = c->Hl[l];
    a.Wc = c->Wcl[l];
    a.Wp = c->Wl[lp];
    a.Hp = c->Hl[lp];
    a.Wcp = c->Wcl[lp];
    a.npix = (uint32_t)a.H * (uint32_t)a.Wc;
    // floor(n / Wc) == umulhi(n, ceil(2^32 / Wc)) for every n < npix when (npix-1) * Wc < 2^32
    a.magic = 0;
    if (a.Wc > 1 && (unsigned long long)(a.npix - 1) * (unsigned long long)a.Wc < (1ull << 32))
        a.magic = (uint32_t)(((1ull << 32) + (unsigned long long)a.Wc - 1) / (unsigned long long)a.Wc);
    a.L = c->L;
    a.Lp = c->Lp;
    a.nch = c->nch;
    a.G = c->G;
    a.log2G = c->log2G;
    a.colour = 0;
    a.plane = (uint32_t)a.H * (uint32_t)a.Wc * (uint32_t)a.Lp;
    a.planep = (uint32_t)a.Hp * (uint32_t)a.Wcp * (uint32_t)a.Lp;
    a.pairD = (size_t)2 * a.plane;
    a.pairM = (size_t)8 * a.plane;
    a.pairMp = (size_t)8 * a.planep;
    a.SS = (uint32_t)c->S | ((uint32_t)c->S << 16);
    a.gl = a.gr = nullptr;
    a.img_elems = 0;
    a.lam = (uint32_t)c->lam_q;
    a.T2d = (uint32_t)c->tau_d | ((uint32_t)c->tau_d << 16);
    a.TT = (uint32_t)c->tau_q | ((uint32_t)c->tau_q << 16);
    return a;
}

}  // namespace

namespace vsbp {
void note_launch(int n) { g_launches += (uint64_t)n; }
}  // namespace vsbp

// Accumulate the pending level timings in FIFO order.  block = 0: only those whose
// end event has already completed (cudaEventQuery; never waits on the device);
// block = 1: all of them (bp_timing_read).
static int timing_drain(vsbp_bp *c, int block)
{
    while (c->n_pending > 0) {
        const int i = c->ev_head;
        if (!block) {
            const cudaError_t q = cudaEventQuery(c->ev[i][1]);
            if (q == cudaErrorNotReady) break;
            CK(q);
        } else {
            CK(cudaEventSynchronize(c->ev[i][1]));
        }
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev[i][0], c->ev[i][1]));
        const int l = c->ev_level[i];
        c->acc_ms[l] += ms;
        c->acc_launches[l] += c->ev_launches[i];
        c->acc_bytes[l] += c->ev_bytes[i];
        c->ev_head = (c->ev_head + 1) % EV_RING;
        --c->n_pending;
    }
    return VSBP_OK;
}

extern "C" {

uint64_t vsbp_launch_count(void) { return g_launches; }

const char *vsbp_strerror(int code)
{
    switch (code) {
    case VSBP_OK: return "ok";
    case VSBP_EINVAL: return "invalid argument";
    case VSBP_EDIM: return "dimension mismatch or workspace too small";
    case VSBP_EOVERFLOW: return "int32 fixed-point bound exceeded";
    case VSBP_ECUDA: return g_errbuf[0] ? g_errbuf : "CUDA error";
    default: return "unknown error";
    }
}

int bp_create(int W, int H, int ndisp, int levels, int iters, float lambda, float data_trunc, float disc_trunc,
              vsbp_bp **out)
{
    if (!out || W < 1 || H < 1 || ndisp < 2 || ndisp > 512 || levels < 1 || levels > 16 || iters < 1)
        return VSBP_EINVAL;
    if (!(lambda >= 0.0f) || !(data_trunc > 0.0f) || !(disc_trunc > 0.0f)) return VSBP_EINVAL;
    if ((long long)W * H > (1ll << 28)) return VSBP_EINVAL;
    const double S = 128.0;  // 2^7, R-6
    const long long lq = rha((double)lambda * S), td = rha((double)data_trunc), tq = rha((double)disc_trunc * S);
    if (td < 1 || tq < 1) return VSBP_EINVAL;
    // R-25: beliefs plus the DT's carry headroom (2^20) must stay below 2^31
    const double bound = (double)lq * (double)td * std::ldexp(1.0, 2 * (levels - 1)) + 4.0 * (double)tq + 1048576.0;
    if (bound >= 2147483648.0) return VSBP_EOVERFLOW;
    vsbp_bp *c = new (std::nothrow) vsbp_bp;
    if (!c) return VSBP_EINVAL;
    memset(c, 0, sizeof *c);
    c->W = W;
    c->H = H;
    c->L = ndisp;
    c->levels = levels;
    c->iters = iters;
    c->lam_q = (int)lq;
    c->tau_d = (int)td;
    c->tau_q = (int)tq;
    c->S = (int)S;
    c->Lp = (ndisp + vsbp::CH - 1) / vsbp::CH * vsbp::CH;
    c->nch = c->Lp / vsbp::CH;
    c->G = 1;
    c->log2G = 0;
    while (c->G < c->nch) {
        c->G <<= 1;
        c->log2G++;
    }
    int w = W, h = H;
    for (int l = 0; l < levels; ++l) {
        c->Wl[l] = w;
        c->Hl[l] = h;
        c->Wcl[l] = (w + 1) / 2;
        c->dbytes[l] = bytes_for_max((long long)c->lam_q * c->tau_d << (2 * l));
        w = (w + 1) / 2;
        h = (h + 1) / 2;
    }
    c->msg_bytes = bytes_for_max(c->tau_q);
    c->dimg = 0;  // measured slower (ALU-bound): DESIGN.md §12
    c->final_fuse = 0;  // measured slower (4x the unpack/sum work per colour-A pixel): DESIGN.md §12
    c->pair_fuse = 1;
    c->pair_band = 64;
    c->pair_min_px = 100000;
    for (int l = 0; l < 16; ++l) {
        c->mcur[l] = 0;
        c->m2_off[l] = 0;
    }
    c->final_ran = 0;
    *out = c;
    return VSBP_OK;
}

int bp_set_option(vsbp_bp *c, int option, int value)
{
    if (!c) return VSBP_EINVAL;
    if (option == VSBP_OPT_MSG_BYTES) {
        const int lossless = bytes_for_max(c->tau_q);
        if (value == 0) value = lossless;
        if (value != 1 && value != 2 && value != 4) return VSBP_EINVAL;
        if (value < lossless) return VSBP_EINVAL;
        c->msg_bytes = value;
        c->ws = nullptr;  // plan changes: workspace must be re-bound
        c->ws_batch = 0;
        return VSBP_OK;
    }
    if (option == VSBP_OPT_KERNEL) {
        if (value < 0 || value > 1) return VSBP_EINVAL;
        c->kernel = value;
        return VSBP_OK;
    }
    if (option == VSBP_OPT_DIMG) {
        if (value < 0 || value > 2) return VSBP_EINVAL;
        c->dimg = value;
        return VSBP_OK;
    }
    if (option == VSBP_OPT_FINAL) {
        if (value < 0 || value > 3) return VSBP_EINVAL;
        c->final_fuse = value;
        return VSBP_OK;
    }
    if (option == VSBP_OPT_PAIR) {
        if (value < 0 || value > 3) return VSBP_EINVAL;
        c->pair_fuse = value;
        c->ws = nullptr;  // plan changes (second message arrays): workspace must be re-bound
        c->ws_batch = 0;
        return VSBP_OK;
    }
    if (option == VSBP_OPT_PAIR_BAND) {
        if (value < 1 || value > 4096) return VSBP_EINVAL;
        c->pair_band = value;
        return VSBP_OK;
    }
    if (option == VSBP_OPT_PAIR_MINPX) {
        if (value < 0) return VSBP_EINVAL;
        c->pair_min_px = value;
        c->ws = nullptr;  // plan changes: workspace must be re-bound
        c->ws_batch = 0;
        return VSBP_OK;
    }
    return VSBP_EINVAL;
}

int bp_get_params(const vsbp_bp *c, int32_t out[8])
{
    if (!c || !out) return VSBP_EINVAL;
    out[0] = c->lam_q;
    out[1] = c->tau_d;
    out[2] = c->tau_q;
    out[3] = c->S;
    out[4] = c->msg_bytes;
    out[5] = c->Lp;
    out[6] = c->levels;
    out[7] = c->iters;
    return VSBP_OK;
}

int bp_level_dims(const vsbp_bp *c, int level, int *W, int *H)
{
    if (!c || !W || !H || level < 0 || level >= c->levels) return VSBP_EINVAL;
    *W = c->Wl[level];
    *H = c->Hl[level];
    return VSBP_OK;
}

size_t bp_workspace_bytes(const vsbp_bp *c, int batch)
{
    if (!c || batch < 1) return 0;
    vsbp_bp tmp = *c;
    plan(&tmp, batch);
    return tmp.total;
}

int bp_set_workspace(vsbp_bp *c, void *dptr, size_t bytes, int batch)
{
    if (!c || !dptr || batch < 1) return VSBP_EINVAL;
    if (((uintptr_t)dptr & 255) != 0) return VSBP_EINVAL;
    plan(c, batch);
    if (bytes < c->total) return VSBP_EDIM;
    c->ws = dptr;
    c->ws_bytes = bytes;
    c->ws_batch = batch;
    return VSBP_OK;
}

int bp_disparity_batch(vsbp_bp *c, int B, const uint8_t *left, const uint8_t *right, int32_t *disp, void *stream)
{
    if (!c || !left || !right || !disp || B < 1) return VSBP_EINVAL;
    if (!c->ws || B > c->ws_batch) return VSBP_EDIM;
    cudaStream_t st = (cudaStream_t)stream;
    if (c->timing) {
        int rc = timing_drain(c, 0);
        // a full ring (thousands of calls without a read) is the one case that waits
        if (!rc && c->n_pending + c->levels > EV_RING) rc = timing_drain(c, 1);
        if (rc) return rc;
    }
    // the workspace is planned for ws_batch pairs: level arrays are [ws_batch][...],
    // a call with B <= ws_batch uses the first B slots (offsets are per-level bases)
    plan(c, c->ws_batch);
    char *ws = wsp(c);
    const int top = c->levels - 1;
    // a1: cost volume, a2: pyramid -- fused for the first F levels when the
    // tile's shared memory fits (costpyr.cu), the rest level by level
    int l_from = 0;
    // levels fused into the cost-volume kernel (tuning knob VSBP_COSTPYR_LEVELS, 1..5)
    static const int fmax = [] {
        const char *e = getenv("VSBP_COSTPYR_LEVELS");
        const int v = e ? atoi(e) : 2;  // measured: 2 fused levels best
        return v < 1 ? 1 : (v > 5 ? 5 : v);
    }();
    const int F = c->levels < fmax ? c->levels : fmax;
    if (c->kernel == 0 && vsbp::costpyr_smem(c->L, c->Lp, F) <= 160 * 1024) {
        vsbp::CostPyrArgs a;
        memset(&a, 0, sizeof a);
        for (int l = 0; l < F; ++l) {
            a.D[l] = ws + c->d_off[l];
            a.dbytes[l] = c->dbytes[l];
            a.W[l] = c->Wl[l];
            a.H[l] = c->Hl[l];
            a.Wc[l] = c->Wcl[l];
            a.pairD[l] = (size_t)2 * c->Hl[l] * c->Wcl[l] * c->Lp;
        }
        a.L = c->L;
        a.Lp = c->Lp;
        a.nch = c->nch;
        a.F = F;
        a.lam_q = c->lam_q;
        a.tau_d = c->tau_d;
        a.write0 = (use_dimg(c) && !dimg_only_singles(c)) ? 0 : 1;  // D_0 is never read when every update computes it
        CK(vsbp::launch_costpyr(left, right, a, B, st));
        l_from = F - 1;
    } else {
        vsbp::Geom g = geom(c, B, 0);
        CK(vsbp::launch_costvol(left, right, ws + c->d_off[0], c->dbytes[0], g, c->lam_q, c->tau_d, st));
    }
    for (int l = l_from; l < top; ++l) {
        vsbp::Geom g = geom(c, B, l);
        CK(vsbp::launch_pyramid(ws + c->d_off[l], c->dbytes[l], ws + c->d_off[l + 1], c->dbytes[l + 1], g, st));
    }
    // a3 + a4, coarse to fine
    for (int l = top; l >= 0; --l) {
        vsbp::Geom g = geom(c, B, l);
        void *D = ws + c->d_off[l];
        c->mcur[l] = 0;
        void *M = msg_base(c, ws, l);
        const void *Mp = (l < top) ? (const void *)msg_base(c, ws, l + 1) : nullptr;
        if (c->iters == 1) {
            // colour 1 is never updated on this level: materialise its initial
            // messages (0 at the top, the parent's otherwise), R-12
            if (l == top) {
                for (int b = 0; b < B; ++b)
                    CK(cudaMemsetAsync(ws + c->m_off[l] + (size_t)b * 8 * g.H * g.Wc * g.Lp * c->msg_bytes, 0,
                                       (size_t)8 * g.H * g.Wc * g.Lp * c->msg_bytes, st));
            } else {
                CK(vsbp::launch_upcopy(M, Mp, c->msg_bytes, g, 1, st));
            }
        }
        const int slot = c->timing ? (c->ev_head + c->n_pending++) % EV_RING : -1;
        if (slot >= 0) CK(cudaEventRecord(c->ev[slot][0], st));
        double bytes = 0.0;
        int launches = 0;
        const bool fast = use_fast(c, l);
        for (int t = 0; t < c->iters; ++t) {
            const int mode = (t > 0) ? 0 : (l == top ? 1 : 2);
            if (fast && use_pair(c, l, B) && t + 1 < c->iters - 1) {
                // iterations t and t+1 in one launch; the level's messages move to its
                // other array (colour t&1's are consumed on chip and never stored)
                vsbp::FastArgs fa = fast_args(c, l, ws, disp);
                fa.colour = (uint32_t)(t & 1);
                CK(vsbp::launch_update_pair(D, c->dbytes[l], fa, B, mode, fast_signed(c, l), pair_band_of(c, l), st));
                c->mcur[l] ^= 1;
                long long nA = 0, nB = 0;
                for (int y = 0; y < g.H; ++y) {
                    nA += (g.W + (((t + y) & 1) ? 0 : 1)) / 2;
                    nB += (g.W + (((t + 1 + y) & 1) ? 0 : 1)) / 2;
                }
                // D of both colours + colour B's 4 messages out (+ its 4 in for MODE 0;
                // the parent's planes once for MODE 2)
                double by = (double)(nA + nB) * c->L * c->dbytes[l] + (double)nB * 4.0 * c->L * c->msg_bytes;
                if (mode == 0) by += (double)nB * 4.0 * c->L * c->msg_bytes;
                if (mode == 2) {
                    const vsbp::Geom gp = geom(c, B, l + 1);
                    by += (double)gp.W * gp.H * 4.0 * c->L * c->msg_bytes;
                }
                bytes += (double)B * by;
                ++launches;
                ++t;  // the pair covered t+1 too
                continue;
            }
            ++launches;
            if (fast) {
                vsbp::FastArgs fa = fast_args(c, l, ws, disp);
                fa.colour = (uint32_t)(t & 1);
                const bool wta = (l == 0 && t == c->iters - 1);  // a5 fused for this colour
                if (wta && use_final(c)) {
                    // last iteration + WTA of both colours, messages not stored
                    if (c->final_fuse == 3)  // row wavefront: A labelled with its update, B from the ring
                        CK(vsbp::launch_update_pair(D, 1, fa, B, 0, fast_signed(c, l), pair_band_of(c, l), st, true));
                    else if (c->final_fuse == 2)
                        CK(vsbp::launch_final_tile(D, fa, B, fast_signed(c, l), st));
                    else
                        CK(vsbp::launch_final_fast(D, fa, B, fast_signed(c, l), st));
                    long long nA = 0, nB = 0;
                    for (int y = 0; y < g.H; ++y) {
                        nA += (g.W + (((t + y) & 1) ? 0 : 1)) / 2;
                        nB += (g.W + (((t + 1 + y) & 1) ? 0 : 1)) / 2;
                    }
                    bytes += (double)B * (nA * (double)c->L * c->dbytes[l] +
                                          nB * ((double)c->L * c->dbytes[l] + 4.0 * c->L * c->msg_bytes));
                    continue;
                }
                int db = c->dbytes[l];
                if (l == 0 && use_dimg(c)) {  // data term from the images, no D_0 read
                    db = 0;
                    fa.gl = left;
                    fa.gr = right;
                    fa.img_elems = (size_t)B * c->W * c->H;
                }
                CK(vsbp::launch_update_fast(D, db, fa, B, mode, wta, fast_signed(c, l), st));
            } else {
                CK(vsbp::launch_update(D, c->dbytes[l], M, Mp, c->msg_bytes, g, mode, t & 1, c->S, c->tau_q, st));
            }
            // pixels of colour t&1: ceil/floor split of each row
            long long npix = 0;
            for (int y = 0; y < g.H; ++y) npix += (g.W + (((t + y) & 1) ? 0 : 1)) / 2;
            if (mode == 2) {
                // first iteration below the top (a3 virtual up-copy): D and the 4 outgoing
                // messages per updated pixel, plus the parent level's message planes read
                // once (4 L bytes per parent pixel; its children read them from L2) --
                // not 4 incoming per child (that undercounts ncu's DRAM by 23 %)
                const vsbp::Geom gp = geom(c, B, l + 1);
                bytes += (double)B * (npix * ((double)c->L * c->dbytes[l] + 4.0 * c->L * c->msg_bytes) +
                                      (double)gp.W * gp.H * 4.0 * c->L * c->msg_bytes);
            } else {
                bytes += (double)B * npix * ((double)c->L * c->dbytes[l] + 8.0 * c->L * c->msg_bytes);
            }
        }
        if (slot >= 0) {
            CK(cudaEventRecord(c->ev[slot][1], st));
            c->ev_level[slot] = l;
            c->ev_launches[slot] = launches;
            c->ev_bytes[slot] = bytes;
        }
    }
    // a5 (the colour updated last was labelled inside its update when the fast kernel ran)
    c->final_ran = use_final(c);
    if (!c->final_ran) {
        if (use_fast(c, 0)) {
            vsbp::FastArgs fa = fast_args(c, 0, ws, disp);
            fa.colour = (uint32_t)(((c->iters - 1) & 1) ^ 1);  // the colour not updated last
            int db = c->dbytes[0];
            if (use_dimg(c)) {
                db = 0;
                fa.gl = left;
                fa.gr = right;
                fa.img_elems = (size_t)B * c->W * c->H;
            }
            CK(vsbp::launch_update_fast(ws + c->d_off[0], db, fa, B, 3, true, false, st));
        } else {
            vsbp::Geom g = geom(c, B, 0);
            CK(vsbp::launch_wta(ws + c->d_off[0], c->dbytes[0], msg_base(c, ws, 0), c->msg_bytes, g, disp, -1, st));
        }
    }
    c->last_B = B;
    c->last_left = left;
    c->last_right = right;
    return VSBP_OK;
}

int bp_disparity(vsbp_bp *c, const uint8_t *left, const uint8_t *right, int32_t *disp, void *stream)
{
    return bp_disparity_batch(c, 1, left, right, disp, stream);
}

int bp_get_messages(vsbp_bp *c, int pair, int level, int32_t *out, void *stream)
{
    if (!c || !out || level < 0 || level >= c->levels || pair < 0) return VSBP_EINVAL;
    if (level == 0 && c->final_ran) return VSBP_EINVAL;  // not materialised (VSBP_OPT_FINAL)
    if (!c->ws || pair >= c->ws_batch) return VSBP_EDIM;
    plan(c, c->ws_batch);
    vsbp::Geom g = geom(c, c->ws_batch, level);
    CK(vsbp::launch_export_msgs(msg_base(c, wsp(c), level), c->msg_bytes, g, pair, out, (cudaStream_t)stream));
    return VSBP_OK;
}

int bp_get_costs(vsbp_bp *c, int pair, int level, int32_t *out, void *stream)
{
    if (!c || !out || level < 0 || level >= c->levels || pair < 0) return VSBP_EINVAL;
    if (!c->ws || pair >= c->ws_batch) return VSBP_EDIM;
    plan(c, c->ws_batch);
    vsbp::Geom g = geom(c, c->ws_batch, level);
    if (level == 0 && use_dimg(c)) {
        // D_0 is not stored on this path (the update computes it): rebuild it from the
        // last call's images (debug/parity only; needs them still alive)
        if (!c->last_left || !c->last_right) return VSBP_EINVAL;
        vsbp::Geom g1 = geom(c, c->last_B, 0);
        CK(vsbp::launch_costvol(c->last_left, c->last_right, wsp(c) + c->d_off[0], c->dbytes[0], g1, c->lam_q,
                                c->tau_d, (cudaStream_t)stream));
    }
    CK(vsbp::launch_export_costs(wsp(c) + c->d_off[level], c->dbytes[level], g, pair, out, (cudaStream_t)stream));
    return VSBP_OK;
}

int bp_timing_enable(vsbp_bp *c, int enable)
{
    if (!c) return VSBP_EINVAL;
    if (enable && !c->timing) {
        for (int i = 0; i < EV_RING; ++i)
            for (int j = 0; j < 2; ++j) CK(cudaEventCreate(&c->ev[i][j]));
        c->ev_head = c->n_pending = 0;
    }
    if (!enable && c->timing) {
        for (int i = 0; i < EV_RING; ++i)
            for (int j = 0; j < 2; ++j) cudaEventDestroy(c->ev[i][j]);
        c->ev_head = c->n_pending = 0;
    }
    c->timing = enable ? 1 : 0;
    return VSBP_OK;
}

int bp_timing_read(vsbp_bp *c, double *ms, int64_t *launches, double *bytes)
{
    if (!c || !ms || !launches || !bytes) return VSBP_EINVAL;
    if (!c->timing) return VSBP_EINVAL;
    int rc = timing_drain(c, 1);
    if (rc) return rc;
    for (int l = 0; l < 16; ++l) {
        ms[l] = c->acc_ms[l];
        launches[l] = c->acc_launches[l];
        bytes[l] = c->acc_bytes[l];
        c->acc_ms[l] = 0.0;
        c->acc_launches[l] = 0;
        c->acc_bytes[l] = 0.0;
    }
    return VSBP_OK;
}

void bp_destroy(vsbp_bp *c)
{
    if (c && c->timing) bp_timing_enable(c, 0);
    delete c;
}

static int jbu_check(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide_rgb, int s, void *disp_hi,
                     float sigma_s, float sigma_r, int radius)
{
    if (B < 1 || !disp_lo || !guide_rgb || !disp_hi || W < 1 || H < 1) return VSBP_EINVAL;
    if (s < 1 || s > 16 || radius < 1 || radius > 8 || !(sigma_s > 0.f) || !(sigma_r > 0.f)) return VSBP_EINVAL;
    if ((long long)W * s * H * s > (1ll << 30)) return VSBP_EINVAL;
    const double r5 = radius + 0.5;
    if (1.4426950408889634 * r5 * r5 / ((double)sigma_s * sigma_s) > 100.0) return VSBP_EINVAL;
    return VSBP_OK;
}

int jbu_upsample_batch(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide_rgb, int s, float *disp_hi,
                       float sigma_s, float sigma_r, int radius, void *stream)
{
    int rc = jbu_check(B, disp_lo, W, H, guide_rgb, s, disp_hi, sigma_s, sigma_r, radius);
    if (rc) return rc;
    CK(vsbp::launch_jbu_fast(B, disp_lo, W, H, guide_rgb, s, disp_hi, sigma_s, sigma_r, radius, nullptr, 1.0f,
                             nullptr, nullptr, (cudaStream_t)stream));
    return VSBP_OK;
}

int jbu_reproject_batch(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide_rgb, int s, float sigma_s,
                        float sigma_r, int radius, const double *Q, float min_disp, float *disp_hi, float *xyz,
                        unsigned long long *n_valid, void *stream)
{
    int rc = jbu_check(B, disp_lo, W, H, guide_rgb, s, disp_hi, sigma_s, sigma_r, radius);
    if (rc) return rc;
    if (!Q || !xyz || !n_valid || !(min_disp > 0.f)) return VSBP_EINVAL;
    float Qf[16];
    for (int i = 0; i < 16; ++i) Qf[i] = (float)Q[i];
    CK(cudaMemsetAsync(n_valid, 0, sizeof(unsigned long long) * (size_t)B, (cudaStream_t)stream));
    CK(vsbp::launch_jbu_fast(B, disp_lo, W, H, guide_rgb, s, disp_hi, sigma_s, sigma_r, radius, Qf, min_disp, xyz,
                             n_valid, (cudaStream_t)stream));
    return VSBP_OK;
}

int jbu_upsample(const int32_t *disp_lo, int W, int H, const uint8_t *guide_rgb, int s, float *disp_hi,
                 float sigma_s, float sigma_r, int radius, void *stream)
{
    return jbu_upsample_batch(1, disp_lo, W, H, guide_rgb, s, disp_hi, sigma_s, sigma_r, radius, stream);
}

int vsbp_q_matrix(double f_du, double f_dv, double u0, double v0, double B, double *Q)
{
    if (!Q || !std::isfinite(f_du) || !std::isfinite(f_dv) || !std::isfinite(u0) || !std::isfinite(v0) ||
        !std::isfinite(B) || f_du == 0.0 ||
        f_dv == 0.0 || B == 0.0)
        return VSBP_EINVAL;
    const double r = f_du / f_dv;
    const double q[16] = {1.0, 0.0, 0.0, -u0, 0.0, r, 0.0, -v0 * r, 0.0, 0.0, 0.0, f_du, 0.0, 0.0, 1.0 / B, 0.0};
    for (int i = 0; i < 16; ++i) Q[i] = q[i];
    return VSBP_OK;
}

size_t compact_workspace_bytes(int B, int W, int H)
{
    if (B < 1 || W < 1 || H < 1) return 0;
    return vsbp::compact_workspace_bytes(B, W, H);
}

int compact_cloud_batch(int B, const float *disp, int W, int H, const double *Q, float min_disp, float *xyz,
                        long long cap_points, long long *offsets, unsigned long long *n_valid, void *workspace,
                        size_t ws_bytes, void *stream)
{
    if (B < 1 || !disp || !Q || !xyz || !offsets || !n_valid || !workspace || W < 1 || H < 1) return VSBP_EINVAL;
    if ((long long)W * H > (1ll << 30) || !(min_disp > 0.f) || cap_points < 0) return VSBP_EINVAL;
    if (ws_bytes < vsbp::compact_workspace_bytes(B, W, H) || ((uintptr_t)workspace & 255)) return VSBP_EINVAL;
    float Qf[16];
    for (int i = 0; i < 16; ++i) Qf[i] = (float)Q[i];
    CK(vsbp::launch_compact(B, disp, W, H, Qf, min_disp, xyz, cap_points, offsets, n_valid, workspace,
                            (cudaStream_t)stream));
    return VSBP_OK;
}

// ---- live timing of the JBU kernel inside jbu_compact_batch (bench.py's second roofline)
namespace {
struct JbuTiming {
    int on = 0, head = 0, n = 0;
    cudaEvent_t ev[64][2];
    double taps[64];
    double ms = 0.0, tap_sum = 0.0;
    long long launches = 0;
    bool created = false;
} g_jt;

int jt_drain(int block)
{
    while (g_jt.n > 0) {
        const int i = g_jt.head;
        if (!block) {
            const cudaError_t q = cudaEventQuery(g_jt.ev[i][1]);
            if (q == cudaErrorNotReady) break;
            CK(q);
        } else {
            CK(cudaEventSynchronize(g_jt.ev[i][1]));
        }
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, g_jt.ev[i][0], g_jt.ev[i][1]));
        g_jt.ms += ms;
        g_jt.tap_sum += g_jt.taps[i];
        ++g_jt.launches;
        g_jt.head = (i + 1) % 64;
        --g_jt.n;
    }
    return VSBP_OK;
}
}  // namespace

int jbu_timing_enable(int enable)
{
    if (enable && !g_jt.created) {
        for (int i = 0; i < 64; ++i)
            for (int k = 0; k < 2; ++k) CK(cudaEventCreate(&g_jt.ev[i][k]));
        g_jt.created = true;
    }
    g_jt.on = enable ? 1 : 0;
    return VSBP_OK;
}

int jbu_timing_read(double *ms, long long *launches, double *taps)
{
    if (!ms || !launches || !taps) return VSBP_EINVAL;
    const int rc = jt_drain(1);
    if (rc) return rc;
    *ms = g_jt.ms;
    *launches = g_jt.launches;
    *taps = g_jt.tap_sum;
    g_jt.ms = g_jt.tap_sum = 0.0;
    g_jt.launches = 0;
    return VSBP_OK;
}

int jbu_compact_batch(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide_rgb, int s, float sigma_s,
                      float sigma_r, int radius, const double *Q, float min_disp, float *disp_hi, float *xyz,
                      long long cap_points, long long *offsets, unsigned long long *n_valid, void *workspace,
                      size_t ws_bytes, void *stream)
{
    int rc = jbu_check(B, disp_lo, W, H, guide_rgb, s, disp_hi, sigma_s, sigma_r, radius);
    if (rc) return rc;
    if (!Q || !xyz || !offsets || !n_valid || !workspace || !(min_disp > 0.f) || cap_points < 0) return VSBP_EINVAL;
    if (ws_bytes < vsbp::compact_workspace_bytes(B, W * s, H * s) || ((uintptr_t)workspace & 255)) return VSBP_EINVAL;
    float Qf[16];
    for (int i = 0; i < 16; ++i) Qf[i] = (float)Q[i];
    cudaStream_t st = (cudaStream_t)stream;
    CK(vsbp::compact_zero_counts(B, W * s, H * s, workspace, st));
    int slot = -1;
    if (g_jt.on) {
        int rc2 = jt_drain(0);
        if (!rc2 && g_jt.n == 64) rc2 = jt_drain(1);
        if (rc2) return rc2;
        slot = (g_jt.head + g_jt.n) % 64;
        CK(cudaEventRecord(g_jt.ev[slot][0], st));
    }
    CK(vsbp::launch_jbu_fast(B, disp_lo, W, H, guide_rgb, s, disp_hi, sigma_s, sigma_r, radius, nullptr, min_disp,
                             nullptr, nullptr, st, vsbp::compact_counts(workspace)));
    if (slot >= 0) {
        CK(cudaEventRecord(g_jt.ev[slot][1], st));
        // the algorithmic work: one weight (one 2^x) per output pixel and window tap
        g_jt.taps[slot] = (double)B * W * s * H * s * (2.0 * radius + 1) * (2.0 * radius + 1);
        ++g_jt.n;
    }
    CK(vsbp::launch_compact_from_counts(B, disp_hi, W * s, H * s, Qf, min_disp, xyz, cap_points, offsets, n_valid,
                                        workspace, st));
    return VSBP_OK;
}

int reproject_batch(int B, const float *disp, int W, int H, const double *Q, float min_disp, float *xyz,
                    unsigned long long *n_valid, void *stream)
{
    if (B < 1 || !disp || !Q || !xyz || !n_valid || W < 1 || H < 1) return VSBP_EINVAL;
    if (!(min_disp > 0.f)) return VSBP_EINVAL;
    if ((long long)W * H > (1ll << 30)) return VSBP_EINVAL;
    float Qf[16];
    for (int i = 0; i < 16; ++i) Qf[i] = (float)Q[i];
    CK(cudaMemsetAsync(n_valid, 0, sizeof(unsigned long long) * (size_t)B, (cudaStream_t)stream));
    CK(vsbp::launch_reproject(B, disp, W, H, Qf, min_disp, xyz, n_valid, (cudaStream_t)stream));
    return VSBP_OK;
}

int reproject(const float *disp, int W, int H, const double *Q, float min_disp, float *xyz,
              unsigned long long *n_valid, void *stream)
{
    return reproject_batch(1, disp, W, H, Q, min_disp, xyz, n_valid, stream);
}

int prep_downsample_batch(int n, const uint8_t *rgb_hi, int W_hi, int H_hi, int s, uint8_t *gray_lo, void *stream)
{
    if (n < 1 || !rgb_hi || !gray_lo || W_hi < 1 || H_hi < 1 || s < 1 || s > 64) return VSBP_EINVAL;
    if (W_hi % s != 0 || H_hi % s != 0) return VSBP_EDIM;
    CK(vsbp::launch_prep(n, rgb_hi, W_hi, H_hi, s, gray_lo, (cudaStream_t)stream));
    return VSBP_OK;
}

int prep_downsample(const uint8_t *rgb_hi, int W_hi, int H_hi, int s, uint8_t *gray_lo, void *stream)
{
    return prep_downsample_batch(1, rgb_hi, W_hi, H_hi, s, gray_lo, stream);
}

int rectify_prep_batch(int n, const uint8_t *rgb_raw, int W_hi, int H_hi, const double *cam, int s,
                       uint8_t *gray_lo, uint8_t *rgb_rect, void *stream)
{
    if (n < 1 || !rgb_raw || !gray_lo || !cam || W_hi < 1 || H_hi < 1 || s < 1 || s > 8) return VSBP_EINVAL;
    if (!(cam[0] > 0.0) || !(cam[1] > 0.0)) return VSBP_EINVAL;
    for (int i = 0; i < 7; ++i)
        if (!std::isfinite(cam[i])) return VSBP_EINVAL;
    if (W_hi % s != 0 || H_hi % s != 0) return VSBP_EDIM;
    if ((long long)W_hi * H_hi > (1ll << 28)) return VSBP_EINVAL;
    if (!vsbp::rectify_domain_ok(W_hi, H_hi, cam)) return VSBP_EOVERFLOW;
    CK(vsbp::launch_rectify_prep(n, rgb_raw, W_hi, H_hi, cam, s, gray_lo, rgb_rect, (cudaStream_t)stream));
    return VSBP_OK;
}

int harris_corners_batch(int n, const uint8_t *gray, int W, int H, int gc, int gr, int K, long long thr,
                         long long *R25, int32_t *xy, long long *resp, int32_t *count, void *stream)
{
    if (n < 1 || !gray || !R25 || !xy || !resp || !count || W < 9 || H < 9 || gc < 1 || gr < 1 || K < 1 || K > 16 ||
        thr < 1)
        return VSBP_EINVAL;
    if ((long long)W * H > (1ll << 28) || (long long)gc * gr > (1ll << 24)) return VSBP_EINVAL;
    CK(vsbp::launch_harris(n, gray, W, H, gc, gr, K, (int64_t)thr, (int64_t *)R25, xy, (int64_t *)resp, count,
                           (cudaStream_t)stream));
    return VSBP_OK;
}

int zssd_match_batch(int n, const uint8_t *img1, const uint8_t *img2, int W, int H, const int32_t *xy,
                     int ncorner, int r, int sr, long long max_cost, int32_t *match, long long *cost, void *stream)
{
    if (n < 1 || !img1 || !img2 || !xy || !match || !cost || W < 1 || H < 1 || ncorner < 0 || r < 1 || r > 7 ||
        sr < 1 || sr > 64 || max_cost < 0)
        return VSBP_EINVAL;
    if ((long long)W * H > (1ll << 28)) return VSBP_EINVAL;
    if (ncorner == 0) return VSBP_OK;
    CK(vsbp::launch_zssd_match(n, img1, img2, W, H, xy, ncorner, r, sr, (int64_t)max_cost, match, (int64_t *)cost,
                               (cudaStream_t)stream));
    return VSBP_OK;
}

size_t icp_workspace_bytes(int ns, int nt) { return (ns < 1 || nt < 1) ? 0 : vsbp::icp_workspace_bytes(ns, nt); }

int icp_register(const float *src, int ns, const float *tgt, int nt, const double *init, int max_iter,
                 double max_dist, double eps, int stride, void *ws, size_t ws_bytes, double *out, void *stream)
{
    if (!src || !tgt || !init || !ws || !out || ns < 1 || nt < 1 || max_iter < 1 || max_iter > 10000 || stride < 1)
        return VSBP_EINVAL;
    if (!(max_dist > 0.0) || !(eps > 0.0) || ((uintptr_t)ws & 255)) return VSBP_EINVAL;
    if (ns > (1 << 28) || nt > (1 << 28)) return VSBP_EINVAL;
    if (ws_bytes < vsbp::icp_workspace_bytes(ns, nt)) return VSBP_EDIM;
    CK(vsbp::launch_icp(src, ns, tgt, nt, init, max_iter, max_dist, eps, stride, ws, out, (cudaStream_t)stream));
    return VSBP_OK;
}

int pair_summary_batch(int B, const int32_t *disp_lo, int W, int H, const unsigned long long *n_valid,
                       uint64_t first_pair_id, vsbp_summary *summary, void *stream)
{
    if (B < 1 || !disp_lo || !summary || W < 1 || H < 1) return VSBP_EINVAL;
    CK(vsbp::launch_summary(B, disp_lo, W, H, n_valid, first_pair_id, summary, (cudaStream_t)stream));
    return VSBP_OK;
}

}  // extern "C"
