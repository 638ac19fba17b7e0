// jbu_fast.cu -- joint bilateral upsampling (a6, Eq.2) fused with the
// reprojection (a7, Eq.3) and the valid-point count, sm_100a.
//
// Eq.2 with R-15..R-19, R-24: for full-res pixel p, taps q in the (2R+1)^2 window
// around c = floor(p/s):  D_p = s * sum_q w_q D'_q / sum_q w_q
//                              = s * (D'_c + sum_q w_q (D'_q - D'_c) / sum_q w_q),
//   log2 w_q = sx[tx] + sy[ty] - cr * (dist2(I_p, I_q) - ref)
// with sx, sy = -log2(e)|p_down - q|^2/(2 sigma_s^2) split per axis (separable),
// cr = log2(e)/(2 sigma_r^2), dist2 = the exact integer squared RGB distance
// (VABSDIFF4 + IDP4A).  The spatial terms depend only on the pixel's sub-position
// (x mod s, y mod s) and the tap offset, so the host tabulates them once per call
// (in double, rounded to f32): sxt[u][t] = sx and ryt[v][t] = 2^sy.  `ref` is any
// per-pixel constant (it cancels in the ratio); it is the centre tap's dist2 when
// cr*that <= 4 (one pass; exponents stay small so the f32 rounding of the exponent
// is tiny), else the window minimum (an extra integer pass).  Out-of-image taps
// get sx = -inf or a row factor of 0 (weight 0): "taps outside the low-res image
// are skipped".  Rows are accumulated separately and scaled by 2^sy at the end.
//
// Accuracy (include/vsbp.h jbu_upsample_batch): the sums accumulate the RESIDUAL
// labels D'_q - D'_c (D'_c = the window centre's label), so the f32 error is
// relative to the label spread of the window, not to the output's magnitude:
// |err| ~ 2e-7 * s * spread full-res px (ex2.approx and rcp.approx are ~2^-22).  A
// window with s * spread > spread_max (256: error <= ~5e-5 px) is computed on the
// PRECISE path instead -- double weights (exp2 in f64) and double sums, one pixel
// at a time (jbu_precise_px).  The test is CTA-uniform first (the staged tile's
// label range, a free by-product of the staging) and per window only inside wide
// tiles, so smooth maps never pay for it.  Both kernels take the same decision per
// window and run the same arithmetic: bit-identical outputs.
//
// Two kernels, the same arithmetic in the same order (bit-identical results):
//  * k_jbu_vec<R,S> (s = S in {2,4,8}): a thread owns P = min(S,4) horizontally
//    adjacent pixels of one footprint row; they share the window, so each tap
//    record is read from shared memory once for P pixels and pixel pairs run on the
//    packed FP32x2 datapath (FADD2/FFMA2).  IDP4A yields the squared distance
//    already as the float bit pattern 2^23 + (dist2 - ref) (accumulator input
//    0x4B000000 + 2^22 - ref).  Per pixel-tap: VABSDIFF4, IDP4A, 1/2 FADD2,
//    1/2 FFMA2, MUFU.EX2, 1/2 FFMA2, 1/2 FADD2 -- the EX2 (16/clk/SM) binds.
//  * k_jbu_fast<R> (any s <= 16, or unaligned buffers): one thread per pixel.
// k_jbu_vec threads own two rows of P pixels (block 32 x 4 threads), k_jbu_fast
// one pixel (32 x 8); both cover a 32P x 8 pixel tile whose low-res taps (guide
// sample + label) are staged once in shared memory as 8-byte records.  The reprojection
// [X Y Z W] = Q [u v D_p 1] follows in registers (one reciprocal of W per pixel);
// one atomic per block counts the points with D_p >= min_disp.
#include <limits.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

// VSBP_JBU_UNROLL_TY: unroll the window's rows in the vector kernel (1: the whole
// (2R+1)^2 x 8-pixel body is straight-line code; 0: one row per loop trip, a 5x
// smaller hot loop for the instruction cache)
#ifndef VSBP_JBU_UNROLL_TY
#define VSBP_JBU_UNROLL_TY 1
#endif
// JB_RP: row passes per CTA of the vector kernel (one staged footprint serves
// JB_RP x JB_Y rows; fewer redundantly staged halo rows per pixel)
#ifndef JB_RP
#define JB_RP 16
#endif
constexpr int JB_X = 32, JB_Y = 8, JB_RMAX = 8, JB_SMAX = 16, JB_TMAX = 2 * JB_RMAX + 1;
constexpr int JB_LW = JB_X + 2 * JB_RMAX + 1, JB_LH = JB_Y + 2 * JB_RMAX + 1;

struct JbuFastArgs {
    int W, H, s;
    float cr;
    float spread_max;             // s * (window label spread) above which the precise path runs
    double cs2, cr2;              // log2(e)/(2 sigma_s^2), log2(e)/(2 sigma_r^2) for the precise path
    int far_thr;                  // centre dist2 above which the window minimum is the reference
    float sxt[JB_SMAX][JB_TMAX];  // [x mod s][tap column]: log2 of the x spatial weight
    float ryt[JB_SMAX][JB_TMAX];  // [y mod s][tap row]: the y spatial weight 2^sy
    float q[16];
    float min_disp;
    int do_xyz;
    // a8 fused counting (jbu_compact_batch): when tile_cnt != null, every pixel with
    // D_p >= min_disp is counted into its compaction segment (128 pixels of a row):
    // tile_cnt[b * pair_segs + y * row_segs + x / 128]
    int *tile_cnt;
    int pair_segs, row_segs;
};

// the valid pixels of one warp row (lane: c pixels of row y; lane 0 at column x0w,
// x grows with the lane) are counted into the compaction segment of x0w: a warp row
// (128, 64 or 32 pixels, aligned to its size) never straddles a segment.  Lane 0 is
// inside whenever any lane is.  Warp-uniform call.
__device__ __forceinline__ void count_row(const JbuFastArgs &a, int b, int y, int x0w, int c, bool inside0)
{
    const int sum = __reduce_add_sync(FULL, c);
    if ((threadIdx.x & 31) == 0 && inside0 && sum)
        atomicAdd(a.tile_cnt + (size_t)b * a.pair_segs + (size_t)y * a.row_segs + (x0w >> 7), sum);
}

__device__ __forceinline__ float ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// stage the block's low-res taps: {guide RGB at the footprint's centre sample, label as f32}.
// Taps outside the low-res image get weight 0 (row factor 0 or column exponent -inf),
// but their record must keep the weighted sums finite: it is a copy of the nearest
// in-image tap (clamped coordinates), which lies in every window that contains the
// phantom, so its colour distance is >= the window minimum and its exponent never
// overflows (0 * inf would be NaN).
// Each warp also leaves the min / max of the labels it staged in wlo / whi[warp]
// (the tile's label range after the barrier, tile_range()).
__device__ __forceinline__ void stage_taps(uint2 *sT, int *wlo, int *whi, const uint8_t *G, const int32_t *Dl, int lx0,
                                           int ly0, int lw, int lh, int s, int Wh, const JbuFastArgs &a, int nthreads)
{
    const int tid = threadIdx.y * JB_X + threadIdx.x;
    int lo = INT_MAX, hi = INT_MIN;
    // (ey, ex) = (e / lw, e % lw) advanced incrementally: two divides per thread
    const int sy = nthreads / lw, sx = nthreads - sy * lw;
    int ey = tid / lw, ex = tid - ey * lw;
    for (int e = tid; e < lw * lh; e += nthreads) {
        const int qy = min(max(ly0 + ey, 0), a.H - 1), qx = min(max(lx0 + ex, 0), a.W - 1);
        ey += sy;
        ex += sx;
        if (ex >= lw) {
            ex -= lw;
            ++ey;
        }
        const uint8_t *g = G + ((size_t)(s * qy + s / 2) * Wh + (size_t)(s * qx + s / 2)) * 3;
        uint2 rec;
        rec.x = (unsigned)g[0] | ((unsigned)g[1] << 8) | ((unsigned)g[2] << 16);
        const int lab = Dl[(size_t)qy * a.W + qx];
        lo = min(lo, lab);
        hi = max(hi, lab);
        rec.y = __float_as_uint((float)lab);
        sT[e] = rec;
    }
    lo = __reduce_min_sync(FULL, lo);
    hi = __reduce_max_sync(FULL, hi);
    if ((threadIdx.x & 31) == 0) {
        wlo[tid >> 5] = lo;
        whi[tid >> 5] = hi;
    }
}

// after the staging barrier: is s * (tile label range) above spread_max?  (CTA-uniform)
__device__ __forceinline__ bool tile_wide(const int *wlo, const int *whi, int nwarps, const JbuFastArgs &a)
{
    int lo = wlo[0], hi = whi[0];
    for (int w = 1; w < nwarps; ++w) {
        lo = min(lo, wlo[w]);
        hi = max(hi, whi[w]);
    }
    return (float)a.s * (float)((long long)hi - lo) > a.spread_max;
}

// the window of (cx, cy) needs the precise path: s * (max - min label over its
// in-image taps) > spread_max (win = the staged window's first record)
template <int R>
__device__ __forceinline__ bool window_wide(const uint2 *win, int lw, int cx, int cy, const JbuFastArgs &a)
{
    float lo = __uint_as_float(win[R * lw + R].y), hi = lo;
#pragma unroll 1
    for (int ty = 0; ty <= 2 * R; ++ty) {
        const int qy = cy - R + ty;
        if (qy < 0 || qy >= a.H) continue;
#pragma unroll 1
        for (int tx = 0; tx <= 2 * R; ++tx) {
            const int qx = cx - R + tx;
            if (qx < 0 || qx >= a.W) continue;
            const float v = __uint_as_float(win[ty * lw + tx].y);
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
        }
    }
    return (float)a.s * (hi - lo) > a.spread_max;
}

// The precise path for one pixel (sub-position u, v of its footprint; colour Ip):
// Eq.2 with double weights w_q = 2^(logit_q - max logit) over the in-image taps
// and double sums of w_q (D'_q - D'_c); the result rounded once to f32.
template <int R>
__device__ __noinline__ float jbu_precise_px(const uint2 *win, int lw, unsigned Ip, int u, int v, int cx, int cy,
                                             const JbuFastArgs &a)
{
    const double fx = ((double)u + 0.5) / a.s - 0.5 + R, fy = ((double)v + 0.5) / a.s - 0.5 + R;
    const double c = (double)__uint_as_float(win[R * lw + R].y);
    double lmax = -INFINITY;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
        double num = 0.0, den = 0.0;
#pragma unroll 1
        for (int ty = 0; ty <= 2 * R; ++ty) {
            const int qy = cy - R + ty;
            if (qy < 0 || qy >= a.H) continue;
#pragma unroll 1
            for (int tx = 0; tx <= 2 * R; ++tx) {
                const int qx = cx - R + tx;
                if (qx < 0 || qx >= a.W) continue;
                const uint2 t = win[ty * lw + tx];
                const unsigned ad = __vabsdiffu4(Ip, t.x);
                const double sx = fx - tx, sy = fy - ty;
                const double logit = -a.cs2 * (sx * sx + sy * sy) - a.cr2 * (double)__dp4a(ad, ad, 0u);
                if (pass == 0) {
                    lmax = fmax(lmax, logit);
                } else {
                    const double w = exp2(logit - lmax);
                    num = fma(w, (double)__uint_as_float(t.y) - c, num);
                    den += w;
                }
            }
        }
        if (pass == 1) return (float)((double)a.s * (c + num / den));
    }
    return 0.f;  // not reached
}

// n / d with one MUFU.RCP (rel. error ~2^-22; the tolerances are 1e-4 px / 1e-5 rel)
__device__ __forceinline__ float fast_div(float n, float d)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    return n * r;
}

// a7 for one pixel: Eq.3 with Q (R-20), NaN below min_disp (R-21).  Row i of
// Q [u v D 1]^T is evaluated as fma(q_i2, D, fma(q_i0, u, fma(q_i1, v, q_i3)))
// in both kernels (the vector kernel does the same on pixel pairs).
__device__ __forceinline__ bool reproject_px(const JbuFastArgs &a, float fu, float fv, float D, float *o)
{
    o[0] = o[1] = o[2] = __int_as_float(0x7fc00000);
    if (!(D >= a.min_disp)) return false;
    float h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = fmaf(a.q[4 * i + 2], D, fmaf(a.q[4 * i], fu, fmaf(a.q[4 * i + 1], fv, a.q[4 * i + 3])));
    const float rW = fast_div(1.0f, h[3]);
    o[0] = h[0] * rW;
    o[1] = h[1] * rW;
    o[2] = h[2] * rW;
    return true;
}

__device__ __forceinline__ void block_count(unsigned *warp_cnt, int cnt, unsigned long long *n_valid, int b,
                                            int nwarps)
{
    cnt = __reduce_add_sync(FULL, cnt);
    if (threadIdx.x == 0) warp_cnt[threadIdx.y] = (unsigned)cnt;
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        unsigned n = 0;
        for (int w = 0; w < nwarps; ++w) n += warp_cnt[w];
        if (n) atomicAdd(n_valid + b, (unsigned long long)n);
    }
}

// ---------------------------------------------------------------- one pixel per thread
template <int R>
__global__ void __launch_bounds__(256) k_jbu_fast(const int32_t *__restrict__ disp_lo, const uint8_t *__restrict__ guide,
                                                  float *__restrict__ disp_hi, float *__restrict__ xyz,
                                                  unsigned long long *__restrict__ n_valid,
                                                  const __grid_constant__ JbuFastArgs a)
{
    constexpr int T = 2 * R + 1;
    __shared__ uint2 sT[JB_LW * JB_LH];
    __shared__ unsigned warp_cnt[JB_Y];
    __shared__ int wlo[JB_Y], whi[JB_Y];
    const int b = blockIdx.z;
    const int s = a.s;
    const int Wh = a.W * s, Hh = a.H * s;
    const int x0 = blockIdx.x * JB_X, y0 = blockIdx.y * JB_Y;
    const int lx0 = x0 / s - R, ly0 = y0 / s - R;
    const int lw = min(x0 + JB_X - 1, Wh - 1) / s + R - lx0 + 1;
    const int lh = min(y0 + JB_Y - 1, Hh - 1) / s + R - ly0 + 1;
    const uint8_t *G = guide + (size_t)b * Hh * Wh * 3;
    stage_taps(sT, wlo, whi, G, disp_lo + (size_t)b * a.H * a.W, lx0, ly0, lw, lh, s, Wh, a, JB_X * JB_Y);
    __syncthreads();
    const bool wide = tile_wide(wlo, whi, JB_Y, a);
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    const bool inside = x < Wh && y < Hh;
    float Dp = 0.f;
    if (inside) {
        const uint8_t *gp = G + ((size_t)y * Wh + x) * 3;
        const unsigned Ip = (unsigned)gp[0] | ((unsigned)gp[1] << 8) | ((unsigned)gp[2] << 16);
        const int cx = x / s, cy = y / s;
        const int u = x - cx * s, v = y - cy * s;
        float sxl[T], rfl[T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int qx = cx - R + t, qy = cy - R + t;
            sxl[t] = (qx >= 0 && qx < a.W) ? a.sxt[u][t] : -INFINITY;
            rfl[t] = (qy >= 0 && qy < a.H) ? a.ryt[v][t] : 0.f;
        }
        const int e0 = (cy - R - ly0) * lw + (cx - R - lx0);
        const float cf = __uint_as_float(sT[e0 + R * lw + R].y);
        if (wide && window_wide<R>(sT + e0, lw, cx, cy, a)) {
            Dp = jbu_precise_px<R>(sT + e0, lw, Ip, u, v, cx, cy, a);
        } else {
        const unsigned ad = __vabsdiffu4(Ip, sT[e0 + R * lw + R].x);
        int ref = (int)__dp4a(ad, ad, 0u);
        if (ref > a.far_thr) {
            // the centre is far in colour: reference the window minimum instead
#pragma unroll
            for (int ty = 0; ty < T; ++ty) {
                if (rfl[ty] == 0.f) continue;
                for (int tx = 0; tx < T; ++tx) {
                    const int qx = cx - R + tx;
                    if (qx < 0 || qx >= a.W) continue;
                    const unsigned adq = __vabsdiffu4(Ip, sT[e0 + ty * lw + tx].x);
                    ref = min(ref, (int)__dp4a(adq, adq, 0u));
                }
            }
        }
        // exact float of (dist2 - ref) via the 2^23 magic: |dist2 - ref| < 2^22
        const unsigned acc = 0x4B000000u + (1u << 22) - (unsigned)ref;
        float num = 0.f, den = 0.f;
#pragma unroll
        for (int ty = 0; ty < T; ++ty) {
            float nr = 0.f, dr = 0.f;
#pragma unroll
            for (int tx = 0; tx < T; ++tx) {
                const uint2 t = sT[e0 + ty * lw + tx];
                const unsigned adq = __vabsdiffu4(Ip, t.x);
                const float f = __uint_as_float(__dp4a(adq, adq, acc)) - 12582912.0f;  // = dist2 - ref
                const float w = ex2(fmaf(-a.cr, f, sxl[tx]));
                nr = fmaf(w, __uint_as_float(t.y) - cf, nr);
                dr += w;
            }
            num = fmaf(rfl[ty], nr, num);
            den = fmaf(rfl[ty], dr, den);
        }
        Dp = (float)s * (cf + fast_div(num, den));
        }
        disp_hi[((size_t)b * Hh + y) * Wh + x] = Dp;
    }
    if (a.tile_cnt)
        count_row(a, b, y, x0, (inside && Dp >= a.min_disp) ? 1 : 0, x0 < Wh && y < Hh);  // warp row: 32 px from x0
    if (!a.do_xyz) return;
    float o[3];
    const bool valid = inside && reproject_px(a, (float)x, (float)y, Dp, o);
    if (inside) {
        float *dst = xyz + (((size_t)b * Hh + y) * Wh + x) * 3;
        dst[0] = o[0];
        dst[1] = o[1];
        dst[2] = o[2];
    }
    block_count(warp_cnt, valid ? 1 : 0, n_valid, b, JB_Y);
}

// ---------------------------------------------------------------- P pixels per thread
typedef unsigned long long f2_t;  // two f32 in one 64-bit register pair

__device__ __forceinline__ f2_t pk2(float a, float b)
{
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(f2_t v, float &a, float &b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c)
{
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b)
{
    f2_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// a thread's P guide pixels of one row: raw() issues the loads (3 words), split()
// turns them into P packed RGB values -- separate, so the vector kernel can fetch the
// next row pass's guide while it computes this one (the loads' latency hidden)
template <int P> struct GuideVec;
template <> struct GuideVec<4> {  // 12 bytes, 4-byte aligned (x % 4 == 0)
    static __device__ __forceinline__ void raw(const uint8_t *g, unsigned w[3])
    {
        const unsigned *p = reinterpret_cast<const unsigned *>(g);
        w[0] = __ldg(p), w[1] = __ldg(p + 1), w[2] = __ldg(p + 2);
    }
    static __device__ __forceinline__ void split(const unsigned w[3], unsigned I[4])
    {
        I[0] = w[0] & 0xFFFFFFu;
        I[1] = __funnelshift_r(w[0], w[1], 24) & 0xFFFFFFu;
        I[2] = __funnelshift_r(w[1], w[2], 16) & 0xFFFFFFu;
        I[3] = w[2] >> 8;
    }
    static __device__ __forceinline__ void load(const uint8_t *g, unsigned I[4])
    {
        unsigned w[3];
        raw(g, w);
        split(w, I);
    }
};
template <> struct GuideVec<2> {  // 6 bytes, 2-byte aligned
    static __device__ __forceinline__ void raw(const uint8_t *g, unsigned w[3])
    {
        const unsigned short *h = reinterpret_cast<const unsigned short *>(g);
        w[0] = __ldg(h), w[1] = __ldg(h + 1), w[2] = __ldg(h + 2);
    }
    static __device__ __forceinline__ void split(const unsigned w[3], unsigned I[2])
    {
        I[0] = w[0] | ((w[1] & 0xFFu) << 16);
        I[1] = (w[1] >> 8) | (w[2] << 8);
    }
    static __device__ __forceinline__ void load(const uint8_t *g, unsigned I[2])
    {
        unsigned w[3];
        raw(g, w);
        split(w, I);
    }
};
#ifndef VSBP_JBU_GPREF
#define VSBP_JBU_GPREF 1  // vector kernel: guide of row pass rp + 1 loaded during pass rp
#endif

template <int R, int S, int NR, int P>
#ifndef VSBP_JBU_MINB
// resident CTAs per SM for the 2-row, 4-pixel variant (the bench's s = 4): 4 leaves
// 128 registers, room for the next row pass's guide words (5: 96, spills)
#define VSBP_JBU_MINB 4
#endif
__global__ void __launch_bounds__(JB_X * JB_Y / NR, NR == 2 ? (P == 4 ? VSBP_JBU_MINB : 8) : (P == 4 ? 3 : 4)) k_jbu_vec(const int32_t *__restrict__ disp_lo,
                                                           const uint8_t *__restrict__ guide,
                                                           float *__restrict__ disp_hi, float *__restrict__ xyz,
                                                           unsigned long long *__restrict__ n_valid,
                                                           const __grid_constant__ JbuFastArgs a)
{
    constexpr int T = 2 * R + 1;
    static_assert(S % P == 0, "a thread's P pixels must share one footprint");
    // NR rows per thread: rows 2t, 2t+1 of a tile are in one footprint row pair (S even)
    constexpr int NT = JB_X * JB_Y / NR;
    // the staged footprint of the CTA's JB_X P x JB_Y JB_RP pixels (sized
    // from JB_RP, R and S, not from the scalar kernel's array)
    constexpr int VLW = (JB_X * P) / S + 2 * R + 1, VLH = (JB_Y * JB_RP + S - 1) / S + 2 * R + 1;
    __shared__ uint2 sT[VLW * VLH];
    __shared__ unsigned warp_cnt[NT / 32];
    __shared__ int wlo[NT / 32], whi[NT / 32];
    const int b = blockIdx.z;
    const int Wh = a.W * S, Hh = a.H * S;
    const int x0 = blockIdx.x * (JB_X * P), y0 = blockIdx.y * (JB_Y * JB_RP);
    const int lx0 = x0 / S - R, ly0 = y0 / S - R;
    const int lw = min(x0 + JB_X * P - 1, Wh - 1) / S + R - lx0 + 1;
    const int lh = min(y0 + JB_Y * JB_RP - 1, Hh - 1) / S + R - ly0 + 1;
    const uint8_t *G = guide + (size_t)b * Hh * Wh * 3;
    stage_taps(sT, wlo, whi, G, disp_lo + (size_t)b * a.H * a.W, lx0, ly0, lw, lh, S, Wh, a, NT);
    __syncthreads();
    const bool wide = tile_wide(wlo, whi, NT / 32, a);
    const int x = x0 + P * threadIdx.x;
    int cnt = 0;
    // per-thread constants of every row pass: the column's x spatial exponents (with
    // out-of-image columns at -inf) and the row sub-position's y factors (JB_Y is a
    // multiple of S, so v0 is the same in every pass)
    const int cx = x / S;
    const int u0 = S == P ? 0 : x - cx * S;
    const int v0 = (y0 + NR * threadIdx.y) % S;
    f2_t sx2[P / 2][T];
#if VSBP_JBU_UNROLL_TY
    float ryv[NR][T];
#endif
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const int qx = cx - R + t;
        const bool okx = qx >= 0 && qx < a.W;
#pragma unroll
        for (int j = 0; j < P / 2; ++j)
            sx2[j][t] = okx ? pk2(a.sxt[u0 + 2 * j][t], a.sxt[u0 + 2 * j + 1][t]) : pk2(-INFINITY, -INFINITY);
#if VSBP_JBU_UNROLL_TY
#pragma unroll
        for (int r = 0; r < NR; ++r) ryv[r][t] = a.ryt[v0 + r][t];
#endif
    }
    unsigned gw[NR][3];  // VSBP_JBU_GPREF: the raw guide words of the next row pass
    // row-pass cursors (advanced by JB_Y rows per pass, no per-pass 64-bit index math):
    // the next pass's guide pixels and this pass's output row
    const size_t grow = (size_t)Wh * 3;
    const uint8_t *gnext = G + ((size_t)(y0 + NR * threadIdx.y) * Wh + x) * 3;
    float *dcur = disp_hi + ((size_t)b * Hh + y0 + NR * threadIdx.y) * Wh + x;
    if (VSBP_JBU_GPREF) {
        const int yb = y0 + NR * threadIdx.y;
#pragma unroll
        for (int r = 0; r < NR; ++r)
            if (x < Wh && yb < Hh) GuideVec<P>::raw(gnext + r * grow, gw[r]);
        gnext += (size_t)JB_Y * grow;
    }
#pragma unroll 1
    for (int rp = 0; rp < JB_RP; ++rp) {
    const int yb = y0 + rp * JB_Y + NR * threadIdx.y;
    const bool inside = x < Wh && yb < Hh;  // Wh % P == 0, Hh % NR == 0: all pixels or none
    const bool inside0 = x0 < Wh && yb < Hh;  // the warp row's first pixel (lane 0)
    float *const drow = dcur;  // this pass's first output row
    dcur += (size_t)JB_Y * Wh;
    unsigned Ipf[NR][P];
    if (VSBP_JBU_GPREF) {
#pragma unroll
        for (int r = 0; r < NR; ++r) GuideVec<P>::split(gw[r], Ipf[r]);
        const int yn = yb + JB_Y;
        if (rp + 1 < JB_RP && x < Wh && yn < Hh) {
#pragma unroll
            for (int r = 0; r < NR; ++r) GuideVec<P>::raw(gnext + r * grow, gw[r]);
        }
        gnext += (size_t)JB_Y * grow;
    }
    float Dp[NR][P];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int k = 0; k < P; ++k) Dp[r][k] = 0.f;
    if (inside) {
        unsigned Ip[NR][P];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            if (VSBP_JBU_GPREF) {
#pragma unroll
                for (int k = 0; k < P; ++k) Ip[r][k] = Ipf[r][k];
            } else {
                GuideVec<P>::load(G + ((size_t)(yb + r) * Wh + x) * 3, Ip[r]);
            }
        }
        const int cy = yb / S;
#if VSBP_JBU_UNROLL_TY
        float rfl[NR][T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int qy = cy - R + t;
            const bool oky = qy >= 0 && qy < a.H;
#pragma unroll
            for (int r = 0; r < NR; ++r) rfl[r][t] = oky ? ryv[r][t] : 0.f;
        }
#endif
        const int e0 = (cy - R - ly0) * lw + (cx - R - lx0);
        const unsigned cen = sT[e0 + R * lw + R].x;
        const float cf = __uint_as_float(sT[e0 + R * lw + R].y);
        if (wide && window_wide<R>(sT + e0, lw, cx, cy, a)) {
#pragma unroll
            for (int r = 0; r < NR; ++r)
#pragma unroll
                for (int k = 0; k < P; ++k) Dp[r][k] = jbu_precise_px<R>(sT + e0, lw, Ip[r][k], u0 + k, v0 + r, cx, cy, a);
        } else {
        int ref[NR][P];
        bool far = false;
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const unsigned ad = __vabsdiffu4(Ip[r][k], cen);
                ref[r][k] = (int)__dp4a(ad, ad, 0u);
                far = far || ref[r][k] > a.far_thr;
            }
        if (far) {
            // some centre is far in colour: that pixel references its window minimum
            // (the window is the same for the thread's NR x P pixels: one pass over the
            // taps, each tap record read once, every pixel's minimum in parallel)
            int m[NR][P];
#pragma unroll
            for (int r = 0; r < NR; ++r)
#pragma unroll
                for (int k = 0; k < P; ++k) m[r][k] = ref[r][k];
#pragma unroll 1
            for (int ty = 0; ty < T; ++ty) {
                if (cy - R + ty < 0 || cy - R + ty >= a.H) continue;
#pragma unroll
                for (int tx = 0; tx < T; ++tx) {
                    const int qx = cx - R + tx;
                    if (qx < 0 || qx >= a.W) continue;
                    const unsigned tq = sT[e0 + ty * lw + tx].x;
#pragma unroll
                    for (int r = 0; r < NR; ++r)
#pragma unroll
                        for (int k = 0; k < P; ++k) {
                            const unsigned adq = __vabsdiffu4(Ip[r][k], tq);
                            m[r][k] = min(m[r][k], (int)__dp4a(adq, adq, 0u));
                        }
                }
            }
#pragma unroll
            for (int r = 0; r < NR; ++r)
#pragma unroll
                for (int k = 0; k < P; ++k)
                    if (ref[r][k] > a.far_thr) ref[r][k] = m[r][k];
        }
        unsigned acc[NR][P];
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int k = 0; k < P; ++k) acc[r][k] = 0x4B000000u + (1u << 22) - (unsigned)ref[r][k];
        const f2_t magic = pk2(-12582912.0f, -12582912.0f);
        const f2_t ncr = pk2(-a.cr, -a.cr);
        f2_t num[NR][P / 2], den[NR][P / 2];
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int j = 0; j < P / 2; ++j) num[r][j] = den[r][j] = 0ull;
#if VSBP_JBU_UNROLL_TY
#pragma unroll
#else
#pragma unroll 1
#endif
        for (int ty = 0; ty < T; ++ty) {
            f2_t nr[NR][P / 2], dr[NR][P / 2];
#pragma unroll
            for (int r = 0; r < NR; ++r)
#pragma unroll
                for (int j = 0; j < P / 2; ++j) nr[r][j] = dr[r][j] = 0ull;
            const uint2 *row = sT + e0 + ty * lw;
#pragma unroll
            for (int tx = 0; tx < T; ++tx) {
                const uint2 tp = row[tx];
                const float dq = __uint_as_float(tp.y) - cf;
                const f2_t dd = pk2(dq, dq);
#pragma unroll
                for (int r = 0; r < NR; ++r)
#pragma unroll
                    for (int j = 0; j < P / 2; ++j) {
                        const unsigned a0 = __vabsdiffu4(Ip[r][2 * j], tp.x), a1 = __vabsdiffu4(Ip[r][2 * j + 1], tp.x);
                        const f2_t F = pk2(__uint_as_float(__dp4a(a0, a0, acc[r][2 * j])),
                                           __uint_as_float(__dp4a(a1, a1, acc[r][2 * j + 1])));
                        const f2_t ex = fma2(ncr, add2(F, magic), sx2[j][tx]);
                        float e0f, e1f;
                        upk2(ex, e0f, e1f);
                        const f2_t w = pk2(ex2(e0f), ex2(e1f));
                        nr[r][j] = fma2(w, dd, nr[r][j]);
                        dr[r][j] = add2(w, dr[r][j]);
                    }
            }
#pragma unroll
            for (int r = 0; r < NR; ++r) {
#if VSBP_JBU_UNROLL_TY
                const f2_t rf2 = pk2(rfl[r][ty], rfl[r][ty]);
#else
                const int qy = cy - R + ty;
                const float rf = (qy >= 0 && qy < a.H) ? a.ryt[v0 + r][ty] : 0.f;
                const f2_t rf2 = pk2(rf, rf);
#endif
#pragma unroll
                for (int j = 0; j < P / 2; ++j) {
                    num[r][j] = fma2(rf2, nr[r][j], num[r][j]);
                    den[r][j] = fma2(rf2, dr[r][j], den[r][j]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < NR; ++r) {
#pragma unroll
            for (int j = 0; j < P / 2; ++j) {
                float n0, n1, d0, d1;
                upk2(num[r][j], n0, n1);
                upk2(den[r][j], d0, d1);
                Dp[r][2 * j] = (float)S * (cf + fast_div(n0, d0));
                Dp[r][2 * j + 1] = (float)S * (cf + fast_div(n1, d1));
            }
        }
        }
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            float *dst = drow + (size_t)r * Wh;
            if (P == 4)
                *reinterpret_cast<float4 *>(dst) = make_float4(Dp[r][0], Dp[r][1], Dp[r][2], Dp[r][3]);
            else
                *reinterpret_cast<float2 *>(dst) = make_float2(Dp[r][0], Dp[r][1]);
        }
    }
    if (a.tile_cnt) {  // a8 counts (all lanes: count_row is warp-collective)
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            int c = 0;
#pragma unroll
            for (int k = 0; k < P; ++k) c += (inside && Dp[r][k] >= a.min_disp) ? 1 : 0;
            count_row(a, b, yb + r, x0, c, inside0);
        }
    }
    if (!a.do_xyz) continue;
    // ---- a7: 3P contiguous floats per thread and row, pixel pairs on FFMA2

    f2_t q2[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) q2[i] = pk2(a.q[i], a.q[i]);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const float fv = (float)(yb + r);
        float o[3 * P];
#pragma unroll
        for (int j = 0; j < P / 2; ++j) {
            const f2_t u2 = pk2((float)(x + 2 * j), (float)(x + 2 * j + 1)), v2 = pk2(fv, fv);
            const f2_t D2 = pk2(Dp[r][2 * j], Dp[r][2 * j + 1]);
            float h[4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const f2_t hi = fma2(q2[4 * i + 2], D2, fma2(q2[4 * i], u2, fma2(q2[4 * i + 1], v2, q2[4 * i + 3])));
                upk2(hi, h[i][0], h[i][1]);
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int k = 2 * j + e;
                const bool valid = inside && Dp[r][k] >= a.min_disp;
                const float rW = fast_div(1.0f, h[3][e]);
                const float nan = __int_as_float(0x7fc00000);
                o[3 * k] = valid ? h[0][e] * rW : nan;
                o[3 * k + 1] = valid ? h[1][e] * rW : nan;
                o[3 * k + 2] = valid ? h[2][e] * rW : nan;
                cnt += valid ? 1 : 0;
            }
        }
        if (inside) {
            float *dst = xyz + (((size_t)b * Hh + yb + r) * Wh + x) * 3;
            if (P == 4) {
                float4 *d4 = reinterpret_cast<float4 *>(dst);
                d4[0] = make_float4(o[0], o[1], o[2], o[3]);
                d4[1] = make_float4(o[4], o[5], o[6], o[7]);
                d4[2] = make_float4(o[8], o[9], o[10], o[11]);
            } else {
                float2 *d2 = reinterpret_cast<float2 *>(dst);
                d2[0] = make_float2(o[0], o[1]);
                d2[1] = make_float2(o[2], o[3]);
                d2[2] = make_float2(o[4], o[5]);
            }
        }
    }
    }
    if (a.do_xyz) block_count(warp_cnt, cnt, n_valid, b, NT / 32);
}

// ---------------------------------------------------------------- launch
// The vector kernel is instantiated for R <= JB_RVEC only (the paper's radii 2..5;
// larger windows take the scalar kernel), two rows per thread and P = min(S, 4)
// pixels per thread: the measured best of P in {2,4} x rows in {1,2}.
// Each extra instantiation costs minutes of ptxas time at full unroll.
constexpr int JB_RVEC = 5;

template <int S, int P>
static void launch_vec(int radius, dim3 grid, cudaStream_t st, const int32_t *disp_lo, const uint8_t *guide,
                       float *disp_hi, float *xyz, unsigned long long *n_valid, const JbuFastArgs &a)
{
    constexpr int NR = 2;
    const dim3 block(JB_X, JB_Y / NR);
    switch (radius) {
    case 1: k_jbu_vec<1, S, NR, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    case 2: k_jbu_vec<2, S, NR, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    case 3: k_jbu_vec<3, S, NR, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    case 4: k_jbu_vec<4, S, NR, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    default: k_jbu_vec<5, S, NR, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    }
}

cudaError_t launch_jbu_fast(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide, int s, float *disp_hi,
                            float sigma_s, float sigma_r, int radius, const float *Qf, float min_disp, float *xyz,
                            unsigned long long *n_valid, cudaStream_t st, int *tile_cnt)
{
    if (s > JB_SMAX || radius > JB_RMAX) return cudaErrorInvalidValue;
    const double log2e = 1.4426950408889634;
    const double cs = log2e / (2.0 * (double)sigma_s * sigma_s);
    JbuFastArgs a;
    memset(&a, 0, sizeof a);
    a.W = W;
    a.H = H;
    a.s = s;
    a.cr = (float)(log2e / (2.0 * (double)sigma_r * sigma_r));
    a.far_thr = (int)floor(4.0 / (double)a.cr);  // reference the minimum when cr * dist2 > ~4
    a.spread_max = 256.0f;
    a.cs2 = cs;
    a.cr2 = log2e / (2.0 * (double)sigma_r * sigma_r);
    // spatial tables (R-15): sub-position u of a footprint has p_down - c = (u + 0.5)/s - 0.5
    for (int u = 0; u < s; ++u) {
        const double f = (u + 0.5) / s - 0.5;
        for (int t = 0; t <= 2 * radius; ++t) {
            const double d = f + (double)(radius - t);
            a.sxt[u][t] = (float)(-cs * d * d);
            a.ryt[u][t] = (float)exp2(-cs * d * d);
        }
    }
    for (int i = 0; i < 16; ++i) a.q[i] = Qf ? Qf[i] : 0.f;
    a.min_disp = min_disp;
    a.do_xyz = xyz != nullptr;
    a.tile_cnt = tile_cnt;
    a.pair_segs = compact_tiles_per_pair(W * s, H * s);
    a.row_segs = compact_segs_per_row(W * s);
    dim3 block(JB_X, JB_Y);
    // the vector kernel needs P-aligned guide words and 4P-byte aligned outputs
    const auto al = [](const void *p, uintptr_t m) { return ((uintptr_t)p & (m - 1)) == 0; };
    const int P = s >= 4 ? 4 : 2;
    const bool vec = (s == 2 || s == 4 || s == 8) && radius <= JB_RVEC && al(guide, P == 4 ? 4 : 2) &&
                     al(disp_hi, 4 * P) && al(xyz, 4 * P);
    if (vec) {
        dim3 grid((W * s + JB_X * P - 1) / (JB_X * P), (H * s + JB_Y * JB_RP - 1) / (JB_Y * JB_RP), B);
        if (s == 2)
            launch_vec<2, 2>(radius, grid, st, disp_lo, guide, disp_hi, xyz, n_valid, a);
        else if (s == 4)
            launch_vec<4, 4>(radius, grid, st, disp_lo, guide, disp_hi, xyz, n_valid, a);
        else
            launch_vec<8, 4>(radius, grid, st, disp_lo, guide, disp_hi, xyz, n_valid, a);
    } else {
        dim3 grid((W * s + JB_X - 1) / JB_X, (H * s + JB_Y - 1) / JB_Y, B);
        switch (radius) {
        case 1: k_jbu_fast<1><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
        case 2: k_jbu_fast<2><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
        case 3: k_jbu_fast<3><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
        case 4: k_jbu_fast<4><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
        case 5: k_jbu_fast<5><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
        case 6: k_jbu_fast<6><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
        case 7: k_jbu_fast<7><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
        default: k_jbu_fast<8><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
        }
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
