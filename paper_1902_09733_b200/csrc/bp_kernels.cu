// bp_kernels.cu -- hierarchical checkerboard min-sum BP on sm_100a (rows a1-a5).
//
//   k_costvol   a1  D_0 = lambda_q * min(|L - R(x-d)|, tau_d)           P:32-34 Eq.1, R-2, R-8
//   k_pyramid   a2  D_{l+1} = sum of existing 2x2 children              P:30 ([4]), R-12
//   k_update    a3+a4  one checkerboard colour of min-sum messages,      P:32-34 Eq.1, R-9..R-12
//                      O(L) truncated-linear distance transform; at t=0
//                      of a level it reads the parent level's messages
//                      directly (virtual up-copy)
//   k_upcopy    a3  materialised up-copy (only needed when iters == 1)   R-12
//   k_wta       a5  argmin_d D_0 + sum of incoming, ties -> smallest d   P:34, R-13
//   k_export_*      int32 natural-layout export for parity tests
//
// Thread mapping (all kernels): one thread = one 16-label chunk of one pixel;
// the G = pow2 >= Lp/16 threads of a pixel are adjacent lanes, so per-label
// reductions and the DT's cross-chunk carries are G-wide warp shuffles.
#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

// ======================================================================== a1
template <typename TD>
__global__ void __launch_bounds__(256) k_costvol(const uint8_t *__restrict__ left, const uint8_t *__restrict__ right,
                                                 TD *__restrict__ D, Geom g, int lam_q, int tau_d)
{
    const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane_g = threadIdx.x & (g.G - 1);
    const long pix = gt >> g.log2G;
    const long per_c = (long)g.H * g.Wc;
    if (lane_g >= g.nch || pix >= (long)g.B * 2 * per_c) return;
    const int b = (int)(pix / (2 * per_c));
    long r = pix - (long)b * 2 * per_c;
    const int c = (int)(r / per_c);
    r -= (long)c * per_c;
    const int y = (int)(r / g.Wc), i = (int)(r - (long)y * g.Wc);
    const int x = 2 * i + ((c + y) & 1);
    if (x >= g.W) return;
    const uint8_t *lrow = left + ((size_t)b * g.H + y) * g.W;
    const uint8_t *rrow = right + ((size_t)b * g.H + y) * g.W;
    const int lv = lrow[x];
    const int border = lam_q * tau_d;
    int v[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
        const int d = lane_g * CH + j;
        int cost = 0;
        if (d < g.L) {
            if (x - d >= 0) {
                int diff = abs(lv - (int)rrow[x - d]);
                cost = lam_q * min(diff, tau_d);
            } else {
                cost = border;
            }
        }
        v[j] = cost;
    }
    Chunk<TD>::store(D + d_off(b, c, y, i, g.H, g.Wc, g.Lp) + lane_g * CH, v);
}

// ======================================================================== a2
template <typename TC, typename TP>
__global__ void __launch_bounds__(256) k_pyramid(const TC *__restrict__ Dc, TP *__restrict__ Dp, Geom g)
{
    // g.W/H/Wc: the CHILD level; g.Wp/Hp/Wcp: the PARENT level being written
    const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane_g = threadIdx.x & (g.G - 1);
    const long pix = gt >> g.log2G;
    const long per_c = (long)g.Hp * g.Wcp;
    if (lane_g >= g.nch || pix >= (long)g.B * 2 * per_c) return;
    const int b = (int)(pix / (2 * per_c));
    long r = pix - (long)b * 2 * per_c;
    const int c = (int)(r / per_c);
    r -= (long)c * per_c;
    const int Y = (int)(r / g.Wcp), I = (int)(r - (long)Y * g.Wcp);
    const int X = 2 * I + ((c + Y) & 1);
    if (X >= g.Wp) return;
    int acc[CH], v[CH];
    zero16(acc);
#pragma unroll
    for (int jy = 0; jy < 2; ++jy)
#pragma unroll
        for (int jx = 0; jx < 2; ++jx) {
            const int x = 2 * X + jx, y = 2 * Y + jy;
            if (x < g.W && y < g.H) {
                Chunk<TC>::load(Dc + d_off(b, (x + y) & 1, y, x >> 1, g.H, g.Wc, g.Lp) + lane_g * CH, v);
#pragma unroll
                for (int j = 0; j < CH; ++j) acc[j] += v[j];
            }
        }
    Chunk<TP>::store(Dp + d_off(b, c, Y, I, g.Hp, g.Wcp, g.Lp) + lane_g * CH, acc);
}

// ======================================================================== a3 + a4
// MODE 0: normal iteration, incoming from this level's field
// MODE 1: first iteration of the top level: all incoming messages are 0
// MODE 2: first iteration of a lower level: incoming read from the parent
//         field, m^l_{q,k} = m^{l+1}_{P(q),k} (R-12; q's neighbour toward p exists)
template <typename TD, typename TM, int MODE>
__global__ void __launch_bounds__(256) k_update(const TD *__restrict__ D, TM *__restrict__ M,
                                                const TM *__restrict__ Mp, Geom g, int colour, int S, int tau_q)
{
    const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane_g = threadIdx.x & (g.G - 1);
    const long pix = gt >> g.log2G;
    const long per_c = (long)g.H * g.Wc;
    bool active = pix < (long)g.B * per_c;
    if (__all_sync(FULL, !active)) return;
    int b = 0, y = 0, i = 0, x = 0;
    if (active) {
        b = (int)(pix / per_c);
        const long r = pix - (long)b * per_c;
        y = (int)(r / g.Wc);
        i = (int)(r - (long)y * g.Wc);
        x = 2 * i + ((colour + y) & 1);
        active = x < g.W;
    }
    const bool io = active && lane_g < g.nch;
    const int d0 = lane_g * CH;
    const int oc = colour ^ 1;  // neighbours' colour
    // neighbour (dx,dy) per direction k and the slot the neighbour uses toward p
    const bool has[4] = {y > 0, y < g.H - 1, x > 0, x < g.W - 1};

    int in[4][CH];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (MODE == 1 || !io || !has[k]) {
            zero16(in[k]);
            continue;
        }
        const int qx = x + (k == 2 ? -1 : (k == 3 ? 1 : 0));
        const int qy = y + (k == 0 ? -1 : (k == 1 ? 1 : 0));
        const int slot = k ^ 1;  // up<->down, left<->right
        if (MODE == 2) {
            const int px = qx >> 1, py = qy >> 1;
            // R-12: the parent's slot toward a missing neighbour counts as 0
            const bool ph = slot == 0 ? py > 0 : slot == 1 ? py < g.Hp - 1 : slot == 2 ? px > 0 : px < g.Wp - 1;
            if (ph)
                Chunk<TM>::load(Mp + m_off(b, (px + py) & 1, slot, py, px >> 1, g.Hp, g.Wcp, g.Lp) + d0, in[k]);
            else
                zero16(in[k]);
        } else {
            Chunk<TM>::load(M + m_off(b, oc, slot, qy, qx >> 1, g.H, g.Wc, g.Lp) + d0, in[k]);
        }
    }
    int tot[CH];
    if (io) {
        Chunk<TD>::load(D + d_off(b, colour, y, i, g.H, g.Wc, g.Lp) + d0, tot);
    } else {
        zero16(tot);
    }
#pragma unroll
    for (int j = 0; j < CH; ++j) tot[j] += in[0][j] + in[1][j] + in[2][j] + in[3][j];

#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int h[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) h[j] = (d0 + j < g.L) ? tot[j] - in[k][j] : BIG;
        // min_d h over the G lanes of this pixel
        int hmin = h[0];
#pragma unroll
        for (int j = 1; j < CH; ++j) hmin = min(hmin, h[j]);
        for (int o = g.G >> 1; o > 0; o >>= 1) hmin = min(hmin, __shfl_xor_sync(FULL, hmin, o, g.G));
        // forward pass f(d) = min(h(d), f(d-1) + S), chunk-local then carried
#pragma unroll
        for (int j = 1; j < CH; ++j) h[j] = min(h[j], h[j - 1] + S);
        int a = h[CH - 1];
        for (int dl = 1; dl < g.G; dl <<= 1) {
            const int v = __shfl_up_sync(FULL, a, dl, g.G);
            if (lane_g >= dl) a = min(a, v + dl * CH * S);
        }
        int cin = __shfl_up_sync(FULL, a, 1, g.G);
        if (lane_g == 0) cin = BIG;
#pragma unroll
        for (int j = 0; j < CH; ++j) h[j] = min(h[j], cin + (j + 1) * S);
        // backward pass g(d) = min(f(d), g(d+1) + S)
#pragma unroll
        for (int j = CH - 2; j >= 0; --j) h[j] = min(h[j], h[j + 1] + S);
        int bb = h[0];
        for (int dl = 1; dl < g.G; dl <<= 1) {
            const int v = __shfl_down_sync(FULL, bb, dl, g.G);
            if (lane_g + dl < g.G) bb = min(bb, v + dl * CH * S);
        }
        int cin2 = __shfl_down_sync(FULL, bb, 1, g.G);
        if (lane_g == g.G - 1) cin2 = BIG;
        const int t = hmin + tau_q;
#pragma unroll
        for (int j = 0; j < CH; ++j) {
            const int gv = min(h[j], cin2 + (CH - j) * S);
            h[j] = (d0 + j < g.L && has[k]) ? min(gv, t) - hmin : 0;
        }
        if (io) Chunk<TM>::store(M + m_off(b, colour, k, y, i, g.H, g.Wc, g.Lp) + d0, h);
    }
}

// ======================================================================== a3 (materialised)
template <typename TM>
__global__ void __launch_bounds__(256) k_upcopy(TM *__restrict__ M, const TM *__restrict__ Mp, Geom g, int colour)
{
    const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane_g = threadIdx.x & (g.G - 1);
    const long pix = gt >> g.log2G;
    const long per_c = (long)g.H * g.Wc;
    if (lane_g >= g.nch || pix >= (long)g.B * per_c) return;
    const int b = (int)(pix / per_c);
    const long r = pix - (long)b * per_c;
    const int y = (int)(r / g.Wc), i = (int)(r - (long)y * g.Wc);
    const int x = 2 * i + ((colour + y) & 1);
    if (x >= g.W) return;
    const bool has[4] = {y > 0, y < g.H - 1, x > 0, x < g.W - 1};
    const int px = x >> 1, py = y >> 1;
    int v[CH];
    const bool phas[4] = {py > 0, py < g.Hp - 1, px > 0, px < g.Wp - 1};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (has[k] && phas[k])
            Chunk<TM>::load(Mp + m_off(b, (px + py) & 1, k, py, px >> 1, g.Hp, g.Wcp, g.Lp) + lane_g * CH, v);
        else
            zero16(v);
        Chunk<TM>::store(M + m_off(b, colour, k, y, i, g.H, g.Wc, g.Lp) + lane_g * CH, v);
    }
}

// ======================================================================== a5
template <typename TD, typename TM>
__global__ void __launch_bounds__(256) k_wta(const TD *__restrict__ D, const TM *__restrict__ M, Geom g,
                                             int32_t *__restrict__ disp, int only_colour)
{
    // only_colour < 0: both colours; else only pixels of that colour
    const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane_g = threadIdx.x & (g.G - 1);
    const long pix = gt >> g.log2G;
    const long per_c = (long)g.H * g.Wc;
    const int ncol = only_colour < 0 ? 2 : 1;
    bool active = pix < (long)g.B * ncol * per_c;
    if (__all_sync(FULL, !active)) return;
    int b = 0, c = 0, y = 0, i = 0, x = 0;
    if (active) {
        b = (int)(pix / (ncol * per_c));
        long r = pix - (long)b * ncol * per_c;
        c = (int)(r / per_c);
        r -= (long)c * per_c;
        if (only_colour >= 0) c = only_colour;
        y = (int)(r / g.Wc);
        i = (int)(r - (long)y * g.Wc);
        x = 2 * i + ((c + y) & 1);
        active = x < g.W;
    }
    const bool io = active && lane_g < g.nch;
    const int d0 = lane_g * CH;
    const bool has[4] = {y > 0, y < g.H - 1, x > 0, x < g.W - 1};
    int e[CH], v[CH];
    if (io)
        Chunk<TD>::load(D + d_off(b, c, y, i, g.H, g.Wc, g.Lp) + d0, e);
    else
        zero16(e);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!io || !has[k]) continue;
        const int qx = x + (k == 2 ? -1 : (k == 3 ? 1 : 0));
        const int qy = y + (k == 0 ? -1 : (k == 1 ? 1 : 0));
        Chunk<TM>::load(M + m_off(b, c ^ 1, k ^ 1, qy, qx >> 1, g.H, g.Wc, g.Lp) + d0, v);
#pragma unroll
        for (int j = 0; j < CH; ++j) e[j] += v[j];
    }
    // key = (belief << 32) | d : the minimum key is the smallest belief, then smallest d
    unsigned long long best = ~0ull;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
        const int d = d0 + j;
        if (io && d < g.L) {
            const unsigned long long key = ((unsigned long long)(unsigned)e[j] << 32) | (unsigned)d;
            best = key < best ? key : best;
        }
    }
    for (int o = g.G >> 1; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(FULL, best, o, g.G);
        best = other < best ? other : best;
    }
    if (active && lane_g == 0) disp[((size_t)b * g.H + y) * g.W + x] = (int32_t)(best & 0xffffffffu);
}

// ======================================================================== exports
template <typename TM>
__global__ void k_export_msgs(const TM *__restrict__ M, Geom g, int b, int32_t *__restrict__ out)
{
    // out: [4][H][W][L] int32, natural layout
    const long n = (long)4 * g.H * g.W * g.L;
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long)gridDim.x * blockDim.x) {
        const int d = (int)(t % g.L);
        long r = t / g.L;
        const int x = (int)(r % g.W);
        r /= g.W;
        const int y = (int)(r % g.H);
        const int k = (int)(r / g.H);
        // slots toward missing neighbours are 0 by definition (R-11); the kernels never read them
        const bool has = k == 0 ? y > 0 : k == 1 ? y < g.H - 1 : k == 2 ? x > 0 : x < g.W - 1;
        out[t] = has ? (int32_t)M[m_off(b, (x + y) & 1, k, y, x >> 1, g.H, g.Wc, g.Lp) + pos_of_label<TM>(d)] : 0;
    }
}

template <typename TD>
__global__ void k_export_costs(const TD *__restrict__ D, Geom g, int b, int32_t *__restrict__ out)
{
    const long n = (long)g.H * g.W * g.L;
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long)gridDim.x * blockDim.x) {
        const int d = (int)(t % g.L);
        long r = t / g.L;
        const int x = (int)(r % g.W);
        const int y = (int)(r / g.W);
        out[t] = (int32_t)D[d_off(b, (x + y) & 1, y, x >> 1, g.H, g.Wc, g.Lp) + pos_of_label<TD>(d)];
    }
}

// ======================================================================== host launchers
static inline unsigned blocks_for(long threads, int bs = 256) { return (unsigned)((threads + bs - 1) / bs); }

#define VSBP_DISPATCH_T(bytes, T, ...)                          \
    switch (bytes) {                                            \
    case 1: { typedef uint8_t T; __VA_ARGS__; } break;          \
    case 2: { typedef uint16_t T; __VA_ARGS__; } break;         \
    default: { typedef int32_t T; __VA_ARGS__; } break;         \
    }

cudaError_t launch_costvol(const uint8_t *left, const uint8_t *right, void *D, int dbytes, const Geom &g, int lam_q,
                           int tau_d, cudaStream_t st)
{
    const long threads = (long)g.B * 2 * g.H * g.Wc * g.G;
    VSBP_DISPATCH_T(dbytes, TD,
                    k_costvol<TD><<<blocks_for(threads), 256, 0, st>>>(left, right, (TD *)D, g, lam_q, tau_d));
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_pyramid(const void *Dc, int cbytes, void *Dp, int pbytes, const Geom &g, cudaStream_t st)
{
    const long threads = (long)g.B * 2 * g.Hp * g.Wcp * g.G;
    VSBP_DISPATCH_T(cbytes, TC,
                    VSBP_DISPATCH_T(pbytes, TP,
                                    k_pyramid<TC, TP><<<blocks_for(threads), 256, 0, st>>>((const TC *)Dc,
                                                                                           (TP *)Dp, g)));
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_update(const void *D, int dbytes, void *M, const void *Mp, int mbytes, const Geom &g, int mode,
                          int colour, int S, int tau_q, cudaStream_t st)
{
    const long threads = (long)g.B * g.H * g.Wc * g.G;
    const unsigned nb = blocks_for(threads);
    VSBP_DISPATCH_T(
        dbytes, TD,
        VSBP_DISPATCH_T(
            mbytes, TM,
            if (mode == 0) k_update<TD, TM, 0><<<nb, 256, 0, st>>>((const TD *)D, (TM *)M, (const TM *)Mp, g,
                                                                   colour, S, tau_q);
            else if (mode == 1) k_update<TD, TM, 1><<<nb, 256, 0, st>>>((const TD *)D, (TM *)M, (const TM *)Mp, g,
                                                                        colour, S, tau_q);
            else k_update<TD, TM, 2><<<nb, 256, 0, st>>>((const TD *)D, (TM *)M, (const TM *)Mp, g, colour, S,
                                                         tau_q);));
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_upcopy(void *M, const void *Mp, int mbytes, const Geom &g, int colour, cudaStream_t st)
{
    const long threads = (long)g.B * g.H * g.Wc * g.G;
    VSBP_DISPATCH_T(mbytes, TM,
                    k_upcopy<TM><<<blocks_for(threads), 256, 0, st>>>((TM *)M, (const TM *)Mp, g, colour));
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_wta(const void *D, int dbytes, const void *M, int mbytes, const Geom &g, int32_t *disp,
                       int only_colour, cudaStream_t st)
{
    const long threads = (long)g.B * (only_colour < 0 ? 2 : 1) * g.H * g.Wc * g.G;
    VSBP_DISPATCH_T(dbytes, TD,
                    VSBP_DISPATCH_T(mbytes, TM,
                                    k_wta<TD, TM><<<blocks_for(threads), 256, 0, st>>>(
                                        (const TD *)D, (const TM *)M, g, disp, only_colour)));
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_export_msgs(const void *M, int mbytes, const Geom &g, int b, int32_t *out, cudaStream_t st)
{
    VSBP_DISPATCH_T(mbytes, TM, k_export_msgs<TM><<<1024, 256, 0, st>>>((const TM *)M, g, b, out));
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_export_costs(const void *D, int dbytes, const Geom &g, int b, int32_t *out, cudaStream_t st)
{
    VSBP_DISPATCH_T(dbytes, TD, k_export_costs<TD><<<1024, 256, 0, st>>>((const TD *)D, g, b, out));
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
