// csbp_api.cu -- the C ABI of row f2 (include/vsbp.h, "Constant-space BP"): context,
// workspace plan and the coarse-to-fine launch sequence.  Host code only.
#include <cmath>
#include <cstring>
#include <new>

#include "vsbp.h"
#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

struct vsbp_csbp {
    int W, H, L, levels, iters, k0;
    int lam_q, tau_d, tau_q, S;
    int Wl[16], Hl[16], kl[16];
    size_t c_off[16], d_off[16], m_off[16], total;
    void *ws;
    int ws_batch;
};

namespace {

long long rha_c(double v) { return v >= 0 ? (long long)std::floor(v + 0.5) : -(long long)std::floor(-v + 0.5); }
size_t al256(size_t v) { return (v + 255) & ~(size_t)255; }

void csbp_plan(vsbp_csbp *c, int batch)
{
    size_t off = 0;
    for (int l = 0; l < c->levels; ++l) {
        const size_t n = (size_t)batch * c->Wl[l] * c->Hl[l] * c->kl[l];
        c->c_off[l] = off;
        off = al256(off + n * sizeof(uint16_t));
        c->d_off[l] = off;
        off = al256(off + n * sizeof(int32_t));
        c->m_off[l] = off;
        off = al256(off + 4 * n * sizeof(int32_t));
    }
    c->total = off;
}

vsbp::CsbpLevel level(const vsbp_csbp *c, int l)
{
    vsbp::CsbpLevel v;
    v.l = l;
    v.W = c->Wl[l];
    v.H = c->Hl[l];
    v.n = v.W * v.H;
    v.k = c->kl[l];
    char *ws = (char *)c->ws;
    v.cand = (uint16_t *)(ws + c->c_off[l]);
    v.dsel = (int32_t *)(ws + c->d_off[l]);
    v.msg = (int32_t *)(ws + c->m_off[l]);
    return v;
}

int cuda_err(cudaError_t) { return VSBP_ECUDA; }

}  // namespace

extern "C" {

int csbp_create(int W, int H, int ndisp, int levels, int iters, int k0, float lambda, float data_trunc,
                float disc_trunc, vsbp_csbp **out)
{
    if (!out || W < 1 || H < 1 || ndisp < 2 || ndisp > 512 || levels < 1 || levels > 16 || iters < 1 || k0 < 1)
        return VSBP_EINVAL;
    if (!(lambda >= 0.0f) || !(data_trunc > 0.0f) || !(disc_trunc > 0.0f)) return VSBP_EINVAL;
    if ((long long)W * H > (1ll << 26)) return VSBP_EINVAL;
    const double S = 128.0;  // R-6
    const long long lq = rha_c((double)lambda * S), td = rha_c((double)data_trunc), tq = rha_c((double)disc_trunc * S);
    if (td < 1 || tq < 1) return VSBP_EINVAL;
    const double bound = (double)lq * (double)td * std::ldexp(1.0, 2 * (levels - 1)) + 4.0 * (double)tq + 1048576.0;
    if (bound >= 2147483648.0) return VSBP_EOVERFLOW;
    vsbp_csbp *c = new (std::nothrow) vsbp_csbp;
    if (!c) return VSBP_EINVAL;
    memset(c, 0, sizeof *c);
    c->W = W;
    c->H = H;
    c->L = ndisp;
    c->levels = levels;
    c->iters = iters;
    c->k0 = k0;
    c->lam_q = (int)lq;
    c->tau_d = (int)td;
    c->tau_q = (int)tq;
    c->S = (int)S;
    int w = W, h = H;
    for (int l = 0; l < levels; ++l) {
        c->Wl[l] = w;
        c->Hl[l] = h;
        const long long k = (long long)k0 << l;
        c->kl[l] = k < ndisp ? (int)k : ndisp;  // R-32
        if (c->kl[l] > vsbp::CS_KMAX) {
            delete c;
            return VSBP_EINVAL;
        }
        w = (w + 1) / 2;
        h = (h + 1) / 2;
    }
    *out = c;
    return VSBP_OK;
}

size_t csbp_workspace_bytes(const vsbp_csbp *c, int batch)
{
    if (!c || batch < 1) return 0;
    vsbp_csbp t = *c;
    csbp_plan(&t, batch);
    return t.total;
}

int csbp_set_workspace(vsbp_csbp *c, void *dptr, size_t bytes, int batch)
{
    if (!c || !dptr || batch < 1 || ((uintptr_t)dptr & 255)) return VSBP_EINVAL;
    csbp_plan(c, batch);
    if (bytes < c->total) return VSBP_EDIM;
    c->ws = dptr;
    c->ws_batch = batch;
    return VSBP_OK;
}

int csbp_disparity_batch(vsbp_csbp *c, int B, const uint8_t *left, const uint8_t *right, int32_t *disp,
                         void *stream)
{
    if (!c || !left || !right || !disp || B < 1) return VSBP_EINVAL;
    if (!c->ws || B > c->ws_batch) return VSBP_EDIM;
    csbp_plan(c, c->ws_batch);
    cudaStream_t st = (cudaStream_t)stream;
    vsbp::CsbpArgs a;
    a.W = c->W;
    a.H = c->H;
    a.L = c->L;
    a.lam_q = c->lam_q;
    a.tau_d = c->tau_d;
    a.tau_q = c->tau_q;
    a.S = c->S;
    const int top = c->levels - 1;
    cudaError_t e;
    for (int l = top; l >= 0; --l) {
        const vsbp::CsbpLevel lv = level(c, l);
        if (l == top)
            e = vsbp::launch_csbp_top(left, right, a, lv, B, st);
        else
            e = vsbp::launch_csbp_init(left, right, a, lv, level(c, l + 1), B, st);
        if (e != cudaSuccess) return cuda_err(e);
        for (int t = 0; t < c->iters; ++t) {
            e = vsbp::launch_csbp_update(a, lv, t & 1, B, st);
            if (e != cudaSuccess) return cuda_err(e);
        }
    }
    e = vsbp::launch_csbp_wta(level(c, 0), disp, B, st);
    if (e != cudaSuccess) return cuda_err(e);
    return VSBP_OK;
}

int csbp_get_candidates(vsbp_csbp *c, int pair, int lev, int32_t *out, void *stream)
{
    if (!c || !out || lev < 0 || lev >= c->levels || pair < 0) return VSBP_EINVAL;
    if (!c->ws || pair >= c->ws_batch) return VSBP_EDIM;
    csbp_plan(c, c->ws_batch);
    const vsbp::CsbpLevel lv = level(c, lev);
    const size_t n = (size_t)lv.n * lv.k;
    cudaError_t e = vsbp::launch_csbp_export(lv.cand + (size_t)pair * n, n, out, (cudaStream_t)stream);
    return e == cudaSuccess ? VSBP_OK : VSBP_ECUDA;
}

void csbp_destroy(vsbp_csbp *c) { delete c; }

}  // extern "C"
