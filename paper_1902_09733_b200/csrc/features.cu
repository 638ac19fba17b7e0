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
//   * k_zssd_match: one CTA per corner stages its patch and the search window in
//     shared memory, evaluates n*ZSSD = n sum (a-b)^2 - (sum a - sum b)^2 at every
//     candidate (exact int32), takes the least cost (ties to raster order), then the
//     least cost beyond Chebyshev distance 2 for the 1.2x ratio gate.
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
constexpr int ZM_T = 256;

__global__ void __launch_bounds__(ZM_T) k_zssd_match(const uint8_t *__restrict__ img1, const uint8_t *__restrict__ img2,
                                                     int W, int H, const int32_t *__restrict__ xy, int ncorner, int r,
                                                     int sr, int64_t max_cost, int32_t *__restrict__ match,
                                                     int64_t *__restrict__ mcost)
{
    extern __shared__ __align__(16) unsigned char zsm[];
    const int b = blockIdx.y, c = blockIdx.x;
    const size_t cs = (size_t)b * ncorner + c;
    const int x = xy[2 * cs], y = xy[2 * cs + 1];
    if (threadIdx.x == 0) {
        match[2 * cs] = match[2 * cs + 1] = -1;
        mcost[cs] = -1;
    }
    if (x < r || y < r || x + r >= W || y + r >= H) return;
    const int P = 2 * r + 1, n = P * P;
    const int S = 2 * sr + 1;          // candidate grid side
    const int RW = S + 2 * r;          // staged img2 window side
    uint8_t *pa = zsm;                 // [P][P]
    uint8_t *rb = zsm + n;             // [RW][RW], out-of-image bytes never used
    unsigned *cost = reinterpret_cast<unsigned *>(zsm + ((n + RW * RW + 15) & ~15));  // [S][S], ~0 = invalid
    const uint8_t *I1 = img1 + (size_t)b * W * H, *I2 = img2 + (size_t)b * W * H;
    for (int e = threadIdx.x; e < n; e += ZM_T) pa[e] = __ldg(I1 + (size_t)(y - r + e / P) * W + (x - r + e % P));
    const int wx0 = x - sr - r, wy0 = y - sr - r;
    for (int e = threadIdx.x; e < RW * RW; e += ZM_T) {
        const int u = wx0 + e % RW, v = wy0 + e / RW;
        rb[e] = (u >= 0 && v >= 0 && u < W && v < H) ? __ldg(I2 + (size_t)v * W + u) : 0;
    }
    __syncthreads();
    int sa = 0;
    for (int e = 0; e < n; ++e) sa += pa[e];
    // costs and the best candidate (cost, raster index) as one 64-bit key
    unsigned long long best = ~0ull;
    for (int e = threadIdx.x; e < S * S; e += ZM_T) {
        const int dy = e / S, dx = e - dy * S;
        const int u = x - sr + dx, v = y - sr + dy;
        unsigned cst = 0xffffffffu;
        if (u >= r && v >= r && u + r < W && v + r < H) {
            int sb = 0, sdd = 0;
            for (int j = 0; j < P; ++j) {
                const uint8_t *ra = pa + j * P, *rr = rb + (dy + j) * RW + dx;
                for (int i = 0; i < P; ++i) {
                    const int bb = rr[i], d = (int)ra[i] - bb;
                    sb += bb;
                    sdd += d * d;
                }
            }
            // n * ZSSD < 2^32 for r <= 7 (225 * 225 * 65025)
            cst = (unsigned)((int64_t)n * sdd - (int64_t)(sa - sb) * (sa - sb));
            const unsigned long long key = ((unsigned long long)cst << 32) | (unsigned)e;
            best = key < best ? key : best;
        }
        cost[e] = cst;
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
    // the least cost beyond Chebyshev distance 2 of the best
    unsigned sec = 0xffffffffu;
    for (int e = threadIdx.x; e < S * S; e += ZM_T) {
        const int dy = e / S, dx = e - dy * S;
        if (abs(dx - bdx) <= 2 && abs(dy - bdy) <= 2) continue;
        sec = min(sec, cost[e]);
    }
    __shared__ unsigned wsec[ZM_T / 32];
    for (int o = 16; o > 0; o >>= 1) sec = min(sec, __shfl_xor_sync(FULL, sec, o));
    __syncthreads();  // wbest reads done before wsec writes share the barrier pattern
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
    const int P = 2 * r + 1, S = 2 * sr + 1, RW = S + 2 * r;
    return (((size_t)P * P + (size_t)RW * RW + 15) & ~(size_t)15) + (size_t)S * S * sizeof(int);
}

cudaError_t launch_zssd_match(int n, const uint8_t *img1, const uint8_t *img2, int W, int H, const int32_t *xy,
                              int ncorner, int r, int sr, int64_t max_cost, int32_t *match, int64_t *mcost,
                              cudaStream_t st)
{
    const size_t smem = zssd_smem(r, sr);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_zssd_match, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k_zssd_match<<<dim3(ncorner, n), ZM_T, smem, st>>>(img1, img2, W, H, xy, ncorner, r, sr, max_cost, match, mcost);
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
