// costpyr.cu -- fused cost volume + the first pyramid levels (rows a1 + a2), sm_100a.
//
// a1: D_0(x,y,d) = lambda_q * min(|L(x,y) - R(x-d,y)|, tau_d), and lambda_q*tau_d
//     where x-d < 0 (Eq.1 E_D; R-2, R-8).
// a2: D_{l+1}(X,Y,d) = sum of the existing children D_l(2X+jx, 2Y+jy, d) (P:30 [4];
//     R-12).  Ceil-halved dimensions make every 16x16-aligned level-0 tile map onto
//     aligned 8x8 / 4x4 / 2x2 / 1x1 tiles of levels 1..4, all children inside it.
//
// One CTA = one 16x16 tile of level-0 pixels of one pair.  It stages the tile's
// left pixels and the right-image span it needs (16 rows x (L+15) bytes) in shared
// memory; one thread computes one 16-label chunk of a 2x2 quad of level-0 pixels
// and sums it into the quad's level-1 chunk in registers; levels 2..F-1 follow
// from the previous level in shared memory (int32), every level written to HBM once in the
// colour-split, chunk-packed layout of vsbp_internal.cuh.  The cost volume is
// never read back from HBM to build the pyramid: HBM traffic is the images plus
// one write of each fused level.
#include <stdlib.h>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

constexpr int CP_T = 16;
#ifndef VSBP_CP_MINB
#define VSBP_CP_MINB 5  // resident CTAs per SM of k_costpyr_fast (48 registers; 4: 6864, 5: 6878, 6: 6875 pairs/s)
#endif  // level-0 tile side (levels 0..4 of a tile nest inside it)

__device__ __forceinline__ void store_chunk(void *base, int bytes, size_t off, const int v[CH])
{
    if (bytes == 1)
        Chunk<uint8_t>::store((uint8_t *)base + off, v);
    else if (bytes == 2)
        Chunk<uint16_t>::store((uint16_t *)base + off, v);
    else
        Chunk<int32_t>::store((int32_t *)base + off, v);
}

// levels 2..F-1 (a2) from the previous level's int32 chunks in shared memory
__device__ __forceinline__ void upper_levels(const CostPyrArgs &a, int *sD, int X0, int Y0, int b)
{
    const int Lp = a.Lp, nch = a.nch;
    int *prev = sD;
    int Tp = CP_T / 2;
    for (int l = 2; l < a.F; ++l) {
        __syncthreads();
        const int T = Tp >> 1;
        int *cur = prev + (size_t)Tp * Tp * Lp;
        const int Wl = a.W[l], Hl = a.H[l], Wcl = a.Wc[l];
        const int Wc_ = a.W[l - 1], Hc_ = a.H[l - 1];
        const int Xl = X0 >> l, Yl = Y0 >> l;
        for (int it = threadIdx.x; it < T * T * nch; it += blockDim.x) {
            const int p = it / nch, k = it - p * nch;
            const int px = p % T, py = p / T;
            const int X = Xl + px, Y = Yl + py;
            int v[CH];
            zero16(v);
            if (X < Wl && Y < Hl) {
#pragma unroll
                for (int jy = 0; jy < 2; ++jy)
#pragma unroll
                    for (int jx = 0; jx < 2; ++jx) {
                        if (2 * X + jx >= Wc_ || 2 * Y + jy >= Hc_) continue;
                        const int4 *src =
                            reinterpret_cast<const int4 *>(prev + (size_t)((2 * py + jy) * Tp + 2 * px + jx) * Lp + k * CH);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int4 w = src[u];
                            v[4 * u] += w.x;
                            v[4 * u + 1] += w.y;
                            v[4 * u + 2] += w.z;
                            v[4 * u + 3] += w.w;
                        }
                    }
                store_chunk(a.D[l], a.dbytes[l],
                            (size_t)b * a.pairD[l] + d_off(0, (X + Y) & 1, Y, X >> 1, Hl, Wcl, Lp) + k * CH, v);
            }
            if (l + 1 < a.F) {
                int4 *dst = reinterpret_cast<int4 *>(cur + (size_t)p * Lp + k * CH);
#pragma unroll
                for (int u = 0; u < 4; ++u) dst[u] = make_int4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
            }
        }
        prev = cur;
        Tp = T;
    }
}

__global__ void __launch_bounds__(256) k_costpyr(const uint8_t *__restrict__ left, const uint8_t *__restrict__ right,
                                                 CostPyrArgs a)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int b = blockIdx.z;
    const int X0 = blockIdx.x * CP_T, Y0 = blockIdx.y * CP_T;
    const int L = a.L, Lp = a.Lp, nch = a.nch;
    const int W = a.W[0], H = a.H[0];
    const int span = CP_T + L - 1;  // right-image columns X0-(L-1) .. X0+15
    uint8_t *sl = smem;                                   // [16][16]
    uint8_t *sr = smem + CP_T * CP_T;                     // [16][span]
    int *sD = reinterpret_cast<int *>(smem + a.img_smem);  // levels 1..F-2, [T_l*T_l][Lp] each
    const uint8_t *lb = left + (size_t)b * H * W;
    const uint8_t *rb = right + (size_t)b * H * W;
    for (int e = threadIdx.x; e < CP_T * CP_T; e += blockDim.x) {
        const int x = X0 + (e & (CP_T - 1)), y = Y0 + e / CP_T;
        sl[e] = (x < W && y < H) ? __ldg(lb + (size_t)y * W + x) : 0;
    }
    for (int e = threadIdx.x; e < CP_T * span; e += blockDim.x) {
        const int r = e / span, j = e - r * span;
        const int x = X0 - (L - 1) + j, y = Y0 + r;
        sr[e] = (x >= 0 && x < W && y < H) ? __ldg(rb + (size_t)y * W + x) : 0;
    }
    __syncthreads();

    // ---- level 0 (a1) and level 1 (a2): one thread = one 16-label chunk of a 2x2
    // quad of level-0 pixels; the quad's sum is its level-1 parent's chunk
    const int border = a.lam_q * a.tau_d;
    constexpr int TQ = CP_T / 2;
    for (int it = threadIdx.x; it < TQ * TQ * nch; it += blockDim.x) {
        const int q = it / nch, k = it - q * nch;
        const int qx = q % TQ, qy = q / TQ;
        int acc[CH];
        zero16(acc);
#pragma unroll
        for (int jy = 0; jy < 2; ++jy)
#pragma unroll
            for (int jx = 0; jx < 2; ++jx) {
                const int px = 2 * qx + jx, py = 2 * qy + jy;
                const int x = X0 + px, y = Y0 + py;
                if (x >= W || y >= H) continue;
                const int lv = sl[py * CP_T + px];
                const uint8_t *rr = sr + py * span + px + (L - 1);  // rr[-d] = R(x-d, y)
                int v[CH];
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    const int d = k * CH + j;
                    int c = 0;
                    if (d < L) c = (x - d >= 0) ? a.lam_q * min(abs(lv - (int)rr[-d]), a.tau_d) : border;
                    v[j] = c;
                    acc[j] += c;
                }
                if (a.write0) store_chunk(a.D[0], a.dbytes[0],
                            (size_t)b * a.pairD[0] + d_off(0, (x + y) & 1, y, x >> 1, H, a.Wc[0], Lp) + k * CH, v);
            }
        if (a.F > 1) {
            const int X = (X0 >> 1) + qx, Y = (Y0 >> 1) + qy;
            if (X < a.W[1] && Y < a.H[1])
                store_chunk(a.D[1], a.dbytes[1],
                            (size_t)b * a.pairD[1] + d_off(0, (X + Y) & 1, Y, X >> 1, a.H[1], a.Wc[1], Lp) + k * CH,
                            acc);
            if (a.F > 2) {
                int4 *dst = reinterpret_cast<int4 *>(sD + (size_t)q * Lp + k * CH);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    dst[u] = make_int4(acc[4 * u], acc[4 * u + 1], acc[4 * u + 2], acc[4 * u + 3]);
            }
        }
    }

    upper_levels(a, sD, X0, Y0, b);
}

// ---------------------------------------------------------------- packed fast path
// Same values as k_costpyr, for parameters where every level-0 cost and every
// level-1 sum fits 16 bits (host check costpyr_fast_ok).  Two labels per 32-bit
// register as s16x2 on the DPX datapath, in the chunk order of vsbp_internal.cuh:
// r_j = (label 16k+j | label 16k+j+8 << 16), which is the u16 storage word j and
// one PRMT away from the u8 storage.  The staged right row holds, per column i,
// the pair (lambda_q R(i), lambda_q R(i-8)) as s16x2, so for a pixel with grey l
//   lambda_q min(|l - r|, tau_d) = max(min((lambda_q l + 1) + ~(lambda_q r), lambda_q tau_d),
//                                      min(-lambda_q l + lambda_q r, lambda_q tau_d))
// (~v = -v-1 per half; the data weight distributes over |.| and min) is two
// VIADDMNMX and a VIMNMX per label pair plus the accumulation.  The two pixels of a
// quad row share 9 of their 16 column reads.  Columns left of the image hold
// -lambda_q tau_d: both mins give lambda_q tau_d there, the border cost (R-8).
// Host check: lambda_q (255 + tau_d) < 2^15, so no half overflows.

__device__ __forceinline__ uint32_t cp_prmt(uint32_t a, uint32_t b, uint32_t sel)
{
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

__device__ __forceinline__ void store_pairs(void *base, int bytes, size_t off, const uint32_t r[8])
{
    if (bytes == 1) {
        uint32_t u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = cp_prmt(r[2 * q], r[2 * q + 1], 0x6240);
        *reinterpret_cast<uint4 *>((uint8_t *)base + off) = make_uint4(u[0], u[1], u[2], u[3]);
    } else {
        uint4 *d = reinterpret_cast<uint4 *>((uint16_t *)base + off);
        d[0] = make_uint4(r[0], r[1], r[2], r[3]);
        d[1] = make_uint4(r[4], r[5], r[6], r[7]);
    }
}

// 32-bit element offset of (colour c, row y, colour-column i) within one pair (the
// per-pair arrays are < 2^32 elements; the pair base is added once in 64 bits)
__device__ __forceinline__ uint32_t d_off32(int c, int y, int i, int H, int Wc, int Lp)
{
    return (((uint32_t)c * (uint32_t)H + (uint32_t)y) * (uint32_t)Wc + (uint32_t)i) * (uint32_t)Lp;
}

// NCH_T > 0: the chunk count is a compile-time power of two (shifts instead of divides).
// TXW: tile width in level-0 pixels (16, or 32 when at most levels 0-1 are fused:
// two quad-chunks per thread amortise the per-thread setup and the staged window)
template <bool PAD, int NCH_T, int TXW = CP_T>
__global__ void __launch_bounds__(256, VSBP_CP_MINB) k_costpyr_fast(const uint8_t *__restrict__ left,
                                                      const uint8_t *__restrict__ right, CostPyrArgs a)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int b = blockIdx.z;
    const int X0 = blockIdx.x * TXW, Y0 = blockIdx.y * CP_T;
    const int L = a.L, Lp = a.Lp, nch = NCH_T > 0 ? NCH_T : a.nch;
    const int W = a.W[0], H = a.H[0];
    const int span = Lp + TXW - 9;         // columns i = X0-Lp+9 .. X0+TXW-1
    const int spanp = (span + 3) & ~3;     // row stride (16-byte rows)
    const int i0 = X0 - Lp + 9;
    uint8_t *sl = smem;                     // [16][TXW]
    uint32_t *sr = reinterpret_cast<uint32_t *>(smem + CP_T * TXW);  // [16][spanp]: lambda_q (R(i), R(i-8)) as s16x2
    int *sD = reinterpret_cast<int *>(smem + a.img_smem);
    const uint8_t *lb = left + (size_t)b * H * W;
    const uint8_t *rb = right + (size_t)b * H * W;
    for (int e = threadIdx.x; e < CP_T * TXW; e += blockDim.x) {
        const int x = X0 + (e & (TXW - 1)), y = Y0 + e / TXW;
        sl[e] = (x < W && y < H) ? __ldg(lb + (size_t)y * W + x) : 0;
    }
    // right rows: one warp per row.  Fast path (W % 4 == 0, 4-byte aligned rows,
    // span + 9 <= 256): every lane issues its (at most two) aligned 32-bit loads of
    // the row window up front and the entries are assembled from them with
    // shuffles, so the warp waits on one load latency instead of a chain of byte
    // loads (the byte loop below was long-scoreboard bound).
    const int lam_i = a.lam_q, sent = -a.lam_q * a.tau_d;
    const int lane = threadIdx.x & 31;
    const bool wpath = (W & 3) == 0 && span + 9 <= 256 && (((uintptr_t)rb) & 3) == 0;
    for (int r = threadIdx.x >> 5; r < CP_T; r += blockDim.x >> 5) {
        const int y = Y0 + r;
        if (y >= H) continue;  // rows below the image are never read
        const uint8_t *rrow = rb + (size_t)y * W;
        if (wpath) {
            const int a0 = i0 - 9;  // multiple of 4: X0 % 16 == 0 and Lp % 16 == 0
            uint32_t w[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = a0 + 4 * (lane + 32 * h);  // words are wholly inside or outside [0, W)
                w[h] = (c >= 0 && c < W && c < i0 + span) ? __ldg(reinterpret_cast<const uint32_t *>(rrow + c)) : 0u;
            }
            for (int jb = 0; jb < span; jb += 32) {  // warp-uniform trip count (shuffles)
                const int j = jb + lane;
                const int i = i0 + j;
                const int b0 = j + 9, b1 = j + 1;  // byte positions of R(i), R(i-8) in the window
                const uint32_t s0l = __shfl_sync(FULL, w[0], (b0 >> 2) & 31), s0h = __shfl_sync(FULL, w[1], (b0 >> 2) & 31);
                const uint32_t s1l = __shfl_sync(FULL, w[0], (b1 >> 2) & 31), s1h = __shfl_sync(FULL, w[1], (b1 >> 2) & 31);
                const uint32_t r0 = ((b0 >> 2) >= 32 ? s0h : s0l) >> (8 * (b0 & 3)) & 0xFFu;
                const uint32_t r1 = ((b1 >> 2) >= 32 ? s1h : s1l) >> (8 * (b1 & 3)) & 0xFFu;
                const int v0 = i < 0 ? sent : (i < W ? lam_i * (int)r0 : 0);
                const int v1 = i - 8 < 0 ? sent : (i - 8 < W ? lam_i * (int)r1 : 0);
                if (j < span) sr[r * spanp + j] = ((uint32_t)v0 & 0xFFFFu) | ((uint32_t)v1 << 16);
            }
        } else {
            for (int j = lane; j < span; j += 32) {
                const int i = i0 + j;
                const int v0 = i < 0 ? sent : (i < W ? lam_i * (int)__ldg(rrow + i) : 0);
                const int v1 = i - 8 < 0 ? sent : (i - 8 < W ? lam_i * (int)__ldg(rrow + i - 8) : 0);
                sr[r * spanp + j] = ((uint32_t)v0 & 0xFFFFu) | ((uint32_t)v1 << 16);
            }
        }
    }
    __syncthreads();

    const uint32_t lt = (uint32_t)(a.lam_q * a.tau_d);
    const uint32_t T2 = lt | (lt << 16);
    constexpr int TQ = CP_T / 2, TQX = TXW / 2;
    uint8_t *D0 = (uint8_t *)a.D[0] + (size_t)b * a.pairD[0] * a.dbytes[0];
    uint8_t *D1 = a.F > 1 ? (uint8_t *)a.D[1] + (size_t)b * a.pairD[1] * a.dbytes[1] : nullptr;
    for (int it = threadIdx.x; it < TQX * TQ * nch; it += blockDim.x) {
        const int q = NCH_T > 0 ? it / NCH_T : it / nch, k = it - q * nch;
        const int qx = q % TQX, qy = q / TQX;
        uint32_t mask[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            mask[j] = PAD ? ((k * CH + j < L ? 0x0000FFFFu : 0u) | (k * CH + j + 8 < L ? 0xFFFF0000u : 0u)) : ~0u;
        uint32_t acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0u;
#pragma unroll
        for (int jy = 0; jy < 2; ++jy) {
            const int py = 2 * qy + jy, y = Y0 + py;
            if (y >= H) continue;
            // columns x0q+1-16k-jj, jj = 0..8: pixel jx=1 uses jj = j, pixel jx=0 uses jj = j+1
            const uint32_t *col = sr + py * spanp + (X0 + 2 * qx + 1 - k * CH - i0);
            uint32_t e[9], ne[9];
#pragma unroll
            for (int jj = 0; jj < 9; ++jj) {
                e[jj] = col[-jj];
                ne[jj] = ~e[jj];
            }
#pragma unroll
            for (int jx = 0; jx < 2; ++jx) {
                const int px = 2 * qx + jx, x = X0 + px;
                if (x >= W) continue;
                const uint32_t lv = (uint32_t)lam_i * sl[py * TXW + px];
                const uint32_t lp1 = (lv + 1u) * 0x00010001u;
                const uint32_t nl2 = ((0u - lv) & 0xFFFFu) * 0x00010001u;
                uint32_t r[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int jj = j + 1 - jx;
                    const uint32_t lo = __viaddmin_s16x2(lp1, ne[jj], T2);  // min(l - r, tau_d)
                    const uint32_t hi = __viaddmin_s16x2(nl2, e[jj], T2);   // min(r - l, tau_d)
                    r[j] = __vmaxs2(lo, hi);
                    if (PAD) r[j] &= mask[j];
                    acc[j] += r[j];
                }
                if (a.write0) store_pairs(D0, a.dbytes[0], d_off32((x + y) & 1, y, x >> 1, H, a.Wc[0], Lp) + k * CH, r);
            }
        }
        if (a.F > 1) {
            const int X = (X0 >> 1) + qx, Y = (Y0 >> 1) + qy;
            if (X < a.W[1] && Y < a.H[1])
                store_pairs(D1, a.dbytes[1], d_off32((X + Y) & 1, Y, X >> 1, a.H[1], a.Wc[1], Lp) + k * CH, acc);
            if (TXW == CP_T && a.F > 2) {
                int4 *dst = reinterpret_cast<int4 *>(sD + (size_t)q * Lp + k * CH);
                dst[0] = make_int4(acc[0] & 0xFFFF, acc[1] & 0xFFFF, acc[2] & 0xFFFF, acc[3] & 0xFFFF);
                dst[1] = make_int4(acc[4] & 0xFFFF, acc[5] & 0xFFFF, acc[6] & 0xFFFF, acc[7] & 0xFFFF);
                dst[2] = make_int4(acc[0] >> 16, acc[1] >> 16, acc[2] >> 16, acc[3] >> 16);
                dst[3] = make_int4(acc[4] >> 16, acc[5] >> 16, acc[6] >> 16, acc[7] >> 16);
            }
        }
    }
    if (TXW == CP_T) upper_levels(a, sD, X0, Y0, b);
}

bool costpyr_fast_ok(const CostPyrArgs &a)
{
    const long long lt = (long long)a.lam_q * a.tau_d;
    if (a.tau_d > 1000 || a.dbytes[0] > 2 || lt > 65535) return false;
    if ((long long)a.lam_q * (255 + a.tau_d) + 1 >= 32768) return false;  // s16 halves of the staged row
    if (a.F > 1 && (a.dbytes[1] > 2 || 4 * lt > 65535)) return false;
    return true;
}

static size_t img_bytes(int L, int Lp)
{
    const size_t generic = (size_t)CP_T * CP_T + (size_t)CP_T * (CP_T + L - 1);
    const size_t fast = (size_t)CP_T * CP_T + (size_t)CP_T * ((Lp + CP_T - 9 + 3) & ~3) * 4;
    const size_t m = generic > fast ? generic : fast;
    return (m + 15) & ~(size_t)15;
}

size_t costpyr_smem(int L, int Lp, int F)
{
    const size_t img = img_bytes(L, Lp);
    size_t px = 0;  // levels 1..F-2 are staged (the last fused level is only written)
    for (int l = 1, T = CP_T / 2; l < F - 1; ++l, T >>= 1) px += (size_t)T * T;
    return img + px * Lp * sizeof(int);
}

cudaError_t launch_costpyr(const uint8_t *left, const uint8_t *right, CostPyrArgs a, int B, cudaStream_t st)
{
    a.img_smem = (int)img_bytes(a.L, a.Lp);
    const size_t smem = costpyr_smem(a.L, a.Lp, a.F);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_costpyr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const void *fs[] = {(const void *)k_costpyr_fast<false, 0>, (const void *)k_costpyr_fast<false, 1>,
                            (const void *)k_costpyr_fast<false, 2>, (const void *)k_costpyr_fast<false, 4>,
                            (const void *)k_costpyr_fast<false, 8>, (const void *)k_costpyr_fast<true, 0>};
        for (const void *f : fs)
            if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((a.W[0] + CP_T - 1) / CP_T, (a.H[0] + CP_T - 1) / CP_T, B);
    // tile width (tuning knob VSBP_COSTPYR_WIDE: 16, 32, 64 or 128 level-0 columns; default 128)
    static const int wide = [] {
        const char *e = getenv("VSBP_COSTPYR_WIDE");
        const int v = e ? atoi(e) : 128;  // measured 16 / 32 / 64 / 128: 7161 / 7198-7273 / 7302-7349 / 7361 pairs/s
        return v >= 128 ? 128 : (v >= 64 ? 64 : (v >= 32 ? 32 : 16));
    }();
    if (wide > CP_T && a.F <= 2 && costpyr_fast_ok(a) && a.L % CH == 0 && a.nch == 4) {
        // 16 x wide tiles: levels 0-1 only (the deeper fused levels need 16 x 16 nesting)
        const size_t simg = ((size_t)CP_T * wide + (size_t)CP_T * ((a.Lp + wide - 9 + 3) & ~3) * 4 + 15) & ~(size_t)15;
        if (a.Lp + wide > 256) return cudaErrorInvalidValue;  // staged window: <= 64 words per row
        a.img_smem = (int)simg;
        dim3 gw((a.W[0] + wide - 1) / wide, (a.H[0] + CP_T - 1) / CP_T, B);
        if (wide == 128)
            k_costpyr_fast<false, 4, 128><<<gw, 256, simg, st>>>(left, right, a);
        else if (wide == 64)
            k_costpyr_fast<false, 4, 64><<<gw, 256, simg, st>>>(left, right, a);
        else
            k_costpyr_fast<false, 4, 32><<<gw, 256, simg, st>>>(left, right, a);
    } else if (costpyr_fast_ok(a) && a.L % CH == 0) {
        switch (a.nch) {
        case 1: k_costpyr_fast<false, 1><<<grid, 256, smem, st>>>(left, right, a); break;
        case 2: k_costpyr_fast<false, 2><<<grid, 256, smem, st>>>(left, right, a); break;
        case 4: k_costpyr_fast<false, 4><<<grid, 256, smem, st>>>(left, right, a); break;
        case 8: k_costpyr_fast<false, 8><<<grid, 256, smem, st>>>(left, right, a); break;
        default: k_costpyr_fast<false, 0><<<grid, 256, smem, st>>>(left, right, a); break;
        }
    } else if (costpyr_fast_ok(a))
        k_costpyr_fast<true, 0><<<grid, 256, smem, st>>>(left, right, a);
    else
        k_costpyr<<<grid, 256, smem, st>>>(left, right, a);
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
