// features.cu -- row f3: Harris corners on a grid + ZSSD matching, sm_100a.
//
// P:48-56 (§2.3, Eq.4-5): "the very fast Harris corner detector", R = det M - k tr^2 M,
// "we choose a patch centered at every Harris corner, and compute correspondence
// between frame I_t1 and I_t2 ... within the given search range ... ZSSD"; P:84:
// "divide the imaging plane to a 30x30 grid and calculate Harris corners inside each
// grid individually".  Readings R-28..R-31 make every step integer:
//   * k_harris: 25 R = 25 (Sxx Syy - Sxy^2) - (Sxx + Syy)^2 in int64, central
//     differences and the 5x5 binomial window, from a shared-memory tile;
//   * k_harris_grid: one CTA per grid cell keeps the K strict 3x3 maxima with the
//     largest response (ties to raster order) -- per-thread sorted lists merged by
//     one warp;
//   * k_zssd_match: one CTA per corner stages the search window in shared memory,
//     evaluates n*ZSSD = n sum (a-b)^2 - (sum a - sum b)^2 at every candidate with
//     packed IDP4A correlation (exact), takes the least cost (ties to raster order),
//     then the least cost beyond Chebyshev distance 2 for the 1.2x ratio gate.
#include <stdint.h>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

constexpr int HR_X = 32, HR_Y = 8, HR_M = 3;  // tile and halo of the response kernel
constexpr int64_t I64MIN = (int64_t)0x8000000000000000ull;

__global__ void __launch_bounds__(256) k_harris(const uint8_t *__restrict__ img, int W, int H,
                                                int64_t *__restrict__ R25)
{
    __shared__ uint8_t sI[HR_Y + 2 * HR_M][HR_X + 2 * HR_M];
    __shared__ int sA[HR_Y + 4][HR_X + 4], sB[HR_Y + 4][HR_X + 4];
    const int b = blockIdx.z;
    const uint8_t *I = img + (size_t)b * W * H;
    const int x0 = blockIdx.x * HR_X, y0 = blockIdx.y * HR_Y;
    const int tid = threadIdx.y * HR_X + threadIdx.x;
    for (int e = tid; e < (HR_Y + 2 * HR_M) * (HR_X + 2 * HR_M); e += HR_X * HR_Y) {
        const int ly = e / (HR_X + 2 * HR_M), lx = e - ly * (HR_X + 2 * HR_M);
        const int x = x0 - HR_M + lx, y = y0 - HR_M + ly;
        sI[ly][lx] = (x >= 0 && y >= 0 && x < W && y < H) ? __ldg(I + (size_t)y * W + x) : 0;
    }
    __syncthreads();
    // derivatives on the tile grown by 2 (the window's reach)
    for (int e = tid; e < (HR_Y + 4) * (HR_X + 4); e += HR_X * HR_Y) {
        const int ly = e / (HR_X + 4), lx = e - ly * (HR_X + 4);
        sA[ly][lx] = (int)sI[ly + 1][lx + 2] - (int)sI[ly + 1][lx];
        sB[ly][lx] = (int)sI[ly + 2][lx + 1] - (int)sI[ly][lx + 1];
    }
    __syncthreads();
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    if (x >= W || y >= H) return;
    int64_t out = I64MIN;
    if (x >= 3 && x <= W - 4 && y >= 3 && y <= H - 4) {
        const int bw[5] = {1, 4, 6, 4, 1};
        int64_t sxx = 0, sxy = 0, syy = 0;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            int rxx = 0, rxy = 0, ryy = 0;  // row sums fit int32: 16 * 65025
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const int A = sA[threadIdx.y + j][threadIdx.x + i], B = sB[threadIdx.y + j][threadIdx.x + i];
                rxx += bw[i] * A * A;
                rxy += bw[i] * A * B;
                ryy += bw[i] * B * B;
            }
            sxx += (int64_t)bw[j] * rxx;
            sxy += (int64_t)bw[j] * rxy;
            syy += (int64_t)bw[j] * ryy;
        }
        out = 25 * (sxx * syy - sxy * sxy) - (sxx + syy) * (sxx + syy);
    }
    R25[(size_t)b * W * H + (size_t)y * W + x] = out;
}

// ---------------------------------------------------------------- grid selection
constexpr int HG_T = 256, HG_KMAX = 16;

// a better than b: larger response, then earlier in raster order
__device__ __forceinline__ bool hg_better(int64_t ra, int ia, int64_t rb, int ib)
{
    return ra > rb || (ra == rb && ia < ib);
}

__global__ void __launch_bounds__(HG_T) k_harris_grid(const int64_t *__restrict__ R25, int W, int H, int gc, int gr,
                                                      int K, int64_t thr, int32_t *__restrict__ out_xy,
                                                      int64_t *__restrict__ resp, int32_t *__restrict__ count)
{
    const int b = blockIdx.y;
    const int cell = blockIdx.x, ci = cell % gc, cj = cell / gc;
    const int x0 = (int)((int64_t)ci * W / gc), x1 = (int)((int64_t)(ci + 1) * W / gc);
    const int y0 = (int)((int64_t)cj * H / gr), y1 = (int)((int64_t)(cj + 1) * H / gr);
    const int cw = x1 - x0, npx = cw * (y1 - y0);
    const int64_t *R = R25 + (size_t)b * W * H;
    // per-thread top-K (K <= HG_KMAX), sorted best first
    int64_t lr[HG_KMAX];
    int li[HG_KMAX];
#pragma unroll
    for (int k = 0; k < HG_KMAX; ++k) {
        lr[k] = I64MIN;
        li[k] = 0x7fffffff;
    }
    for (int e = threadIdx.x; e < npx; e += HG_T) {
        const int y = y0 + e / cw, x = x0 + e % cw;
        if (x < 4 || x > W - 5 || y < 4 || y > H - 5) continue;
        const int64_t r = R[(size_t)y * W + x];
        if (r < thr) continue;
        bool mx = true;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx)
                if ((dx || dy) && R[(size_t)(y + dy) * W + x + dx] >= r) mx = false;
        if (!mx) continue;
        const int idx = y * W + x;
        // sorted insertion; the element pushed past slot K-1 is dropped
        int64_t cr = r;
        int cx = idx;
#pragma unroll
        for (int k = 0; k < HG_KMAX; ++k) {
            if (k < K && hg_better(cr, cx, lr[k], li[k])) {
                const int64_t tr = lr[k];
                const int ti = li[k];
                lr[k] = cr;
                li[k] = cx;
                cr = tr;
                cx = ti;
            }
        }
    }
    // merge: K rounds of a block-wide argmax over the per-thread heads
    __shared__ int64_t wr[HG_T / 32];
    __shared__ int wi[HG_T / 32], wt[HG_T / 32];
    __shared__ int n_found;
    int head = 0;
    if (threadIdx.x == 0) n_found = 0;
    __syncthreads();
    for (int k = 0; k < K; ++k) {
        int64_t r = head < K ? lr[0] : I64MIN;
        int idx = head < K ? li[0] : 0x7fffffff;
        // lr/li are shifted as heads are consumed, so the head is always element 0
        int owner = threadIdx.x;
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t r2 = __shfl_xor_sync(FULL, r, o);
            const int i2 = __shfl_xor_sync(FULL, idx, o);
            const int w2 = __shfl_xor_sync(FULL, owner, o);
            if (hg_better(r2, i2, r, idx)) {
                r = r2;
                idx = i2;
                owner = w2;
            }
        }
        if ((threadIdx.x & 31) == 0) {
            wr[threadIdx.x >> 5] = r;
            wi[threadIdx.x >> 5] = idx;
            wt[threadIdx.x >> 5] = owner;
        }
        __syncthreads();
        int64_t br = wr[0];
        int bi = wi[0], bt = wt[0];
        for (int w = 1; w < HG_T / 32; ++w)
            if (hg_better(wr[w], wi[w], br, bi)) {
                br = wr[w];
                bi = wi[w];
                bt = wt[w];
            }
        const size_t slot = ((size_t)b * gr * gc + cell) * K + k;
        if (threadIdx.x == 0) {
            if (br != I64MIN) {
                out_xy[2 * slot] = bi % W;
                out_xy[2 * slot + 1] = bi / W;
                resp[slot] = br;
                n_found = k + 1;
            } else {
                out_xy[2 * slot] = -1;
                out_xy[2 * slot + 1] = -1;
                resp[slot] = I64MIN;
            }
        }
        if (threadIdx.x == bt && br != I64MIN) {  // pop the owner's head
#pragma unroll
            for (int q = 0; q < HG_KMAX - 1; ++q) {
                lr[q] = lr[q + 1];
                li[q] = li[q + 1];
            }
            lr[HG_KMAX - 1] = I64MIN;
            li[HG_KMAX - 1] = 0x7fffffff;
            ++head;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) count[(size_t)b * gr * gc + cell] = n_found;
}

// ---------------------------------------------------------------- ZSSD matching
// One CTA per corner.  The patch rows of img1 are packed into registers (P bytes per
// row in ceil(P/4) words, zero-padded); the search window of img2 sits in shared
// memory with a row pitch that is a multiple of 4.  A work item is one candidate
// row dy and 4 consecutive dx: per patch row it loads the covering words once and,
// per candidate, aligns them with PRMT and accumulates sum(ab), sum(b), sum(b^2) with
// IDP4A (u8 x u8 -> u32, exact).  n*ZSSD = n (Sa2 - 2 Sab + Sb2) - (Sa - Sb)^2.
constexpr int ZM_T = 256;

template <int R>
__global__ void __launch_bounds__(ZM_T) k_zssd_match(const uint8_t *__restrict__ img1, const uint8_t *__restrict__ img2,
                                                     int W, int H, const int32_t *__restrict__ xy, int ncorner, int sr,
                                                     int64_t max_cost, int32_t *__restrict__ match,
                                                     int64_t *__restrict__ mcost)
{
    constexpr int P = 2 * R + 1, n = P * P, NWP = (P + 3) / 4;  // words per patch row
    extern __shared__ __align__(16) unsigned char zsm[];
    const int b = blockIdx.y, c = blockIdx.x;
    const size_t cs = (size_t)b * ncorner + c;
    const int x = xy[2 * cs], y = xy[2 * cs + 1];
    if (threadIdx.x == 0) {
        match[2 * cs] = match[2 * cs + 1] = -1;
        mcost[cs] = -1;
    }
    if (x < R || y < R || x + R >= W || y + R >= H) return;
    const int S = 2 * sr + 1;                       // candidate grid side
    const int RW = S + 2 * R, RP = (RW + 3 + 8) & ~3;  // staged img2 window, padded pitch
    uint8_t *rb = zsm;                              // [RW][RP]
    unsigned *cost = reinterpret_cast<unsigned *>(zsm + (size_t)RW * RP);  // [S][S], ~0 = invalid
    const uint8_t *I1 = img1 + (size_t)b * W * H, *I2 = img2 + (size_t)b * W * H;
    const int wx0 = x - sr - R, wy0 = y - sr - R;
    for (int e = threadIdx.x; e < RW * RP; e += ZM_T) {
        const int lx = e % RP, ly = e / RP;
        const int u = wx0 + lx, v = wy0 + ly;
        rb[e] = (lx < RW && u >= 0 && v >= 0 && u < W && v < H) ? __ldg(I2 + (size_t)v * W + u) : 0;
    }
    // the patch of img1, packed; sum a and sum a^2
    unsigned pa[P][NWP];
    int sa = 0, sa2 = 0;
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
        for (int q = 0; q < NWP; ++q) {
            unsigned w = 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (4 * q + k < P) {
                    const unsigned v = __ldg(I1 + (size_t)(y - R + j) * W + (x - R + 4 * q + k));
                    w |= v << (8 * k);
                    sa += (int)v;
                    sa2 += (int)(v * v);
                }
            }
            pa[j][q] = w;
        }
    __syncthreads();
    const unsigned lastmask = (P % 4) ? (0xFFFFFFFFu >> (8 * (4 - P % 4))) : 0xFFFFFFFFu;
    const int G4 = (S + 3) / 4;
    unsigned long long best = ~0ull;
    for (int it = threadIdx.x; it < S * G4; it += ZM_T) {
        const int dy = it / G4, dx0 = 4 * (it - dy * G4);
        unsigned sab[4] = {0u, 0u, 0u, 0u}, sb[4] = {0u, 0u, 0u, 0u}, sb2[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const uint8_t *row = rb + (dy + j) * RP + dx0;  // dx0 % 4 == 0, RP % 4 == 0: aligned
            const unsigned *wrow = reinterpret_cast<const unsigned *>(row);
            unsigned w[NWP + 1];
#pragma unroll
            for (int q = 0; q <= NWP; ++q) w[q] = wrow[q];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
#pragma unroll
                for (int q = 0; q < NWP; ++q) {
                    unsigned bw = __byte_perm(w[q], w[q + 1], 0x3210 + 0x1111 * k);
                    if (q == NWP - 1) bw &= lastmask;
                    sab[k] = __dp4a(pa[j][q], bw, sab[k]);
                    sb[k] = __dp4a(0x01010101u, bw, sb[k]);
                    sb2[k] = __dp4a(bw, bw, sb2[k]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int dx = dx0 + k;
            if (dx >= S) break;
            const int u = x - sr + dx, v = y - sr + dy;
            unsigned cst = 0xffffffffu;
            if (u >= R && v >= R && u + R < W && v + R < H) {
                const int64_t sdd = (int64_t)sa2 - 2 * (int64_t)sab[k] + (int64_t)sb2[k];
                const int64_t dm = (int64_t)sa - (int64_t)sb[k];
                cst = (unsigned)((int64_t)n * sdd - dm * dm);  // < 2^32 for R <= 7
                const int e = dy * S + dx;
                const unsigned long long key = ((unsigned long long)cst << 32) | (unsigned)e;
                best = key < best ? key : best;
            }
            cost[dy * S + dx] = cst;
        }
    }
    __shared__ unsigned long long wbest[ZM_T / 32];
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(FULL, best, o);
        best = t < best ? t : best;
    }
    if ((threadIdx.x & 31) == 0) wbest[threadIdx.x >> 5] = best;
    __syncthreads();
    best = wbest[0];
    for (int w = 1; w < ZM_T / 32; ++w) best = wbest[w] < best ? wbest[w] : best;
    if (best == ~0ull) return;
    const int be = (int)(best & 0xffffffffu);
    const unsigned bcost = (unsigned)(best >> 32);
    const int bdy = be / S, bdx = be - bdy * S;
    // the least cost beyond Chebyshev distance 2 of the best (1.2x ratio gate)
    unsigned sec = 0xffffffffu;
    for (int e = threadIdx.x; e < S * S; e += ZM_T) {
        const int dy = e / S, dx = e - dy * S;
        if (abs(dx - bdx) <= 2 && abs(dy - bdy) <= 2) continue;
        sec = min(sec, cost[e]);
    }
    __shared__ unsigned wsec[ZM_T / 32];
    for (int o = 16; o > 0; o >>= 1) sec = min(sec, __shfl_xor_sync(FULL, sec, o));
    if ((threadIdx.x & 31) == 0) wsec[threadIdx.x >> 5] = sec;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned s2 = wsec[0];
        for (int w = 1; w < ZM_T / 32; ++w) s2 = min(s2, wsec[w]);
        const bool ok = (int64_t)bcost <= max_cost && (s2 == 0xffffffffu || 5ll * s2 > 6ll * (long long)bcost);
        if (ok) {
            match[2 * cs] = x - sr + bdx;
            match[2 * cs + 1] = y - sr + bdy;
            mcost[cs] = bcost;
        }
    }
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_harris(int n, const uint8_t *img, int W, int H, int gc, int gr, int K, int64_t thr, int64_t *R25,
                          int32_t *xy, int64_t *resp, int32_t *count, cudaStream_t st)
{
    dim3 g1((W + HR_X - 1) / HR_X, (H + HR_Y - 1) / HR_Y, n);
    k_harris<<<g1, dim3(HR_X, HR_Y), 0, st>>>(img, W, H, R25);
    k_harris_grid<<<dim3(gc * gr, n), HG_T, 0, st>>>(R25, W, H, gc, gr, K, thr, xy, resp, count);
    note_launch(2);
    return cudaGetLastError();
}

size_t zssd_smem(int r, int sr)
{
    const int S = 2 * sr + 1, RW = S + 2 * r, RP = (RW + 3 + 8) & ~3;
    return (size_t)RW * RP + (size_t)S * S * sizeof(unsigned);
}

cudaError_t launch_zssd_match(int n, const uint8_t *img1, const uint8_t *img2, int W, int H, const int32_t *xy,
                              int ncorner, int r, int sr, int64_t max_cost, int32_t *match, int64_t *mcost,
                              cudaStream_t st)
{
    const size_t smem = zssd_smem(r, sr);
    const dim3 grid(ncorner, n);
    cudaError_t e = cudaSuccess;
#define VSBP_Z(R_)                                                                                             \
    case R_:                                                                                                   \
        if (smem > 48 * 1024)                                                                                  \
            e = cudaFuncSetAttribute(k_zssd_match<R_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e == cudaSuccess)                                                                                  \
            k_zssd_match<R_><<<grid, ZM_T, smem, st>>>(img1, img2, W, H, xy, ncorner, sr, max_cost, match, mcost); \
        break;
    switch (r) {
        VSBP_Z(1) VSBP_Z(2) VSBP_Z(3) VSBP_Z(4) VSBP_Z(5) VSBP_Z(6) VSBP_Z(7)
    default: return cudaErrorInvalidValue;
    }
#undef VSBP_Z
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
