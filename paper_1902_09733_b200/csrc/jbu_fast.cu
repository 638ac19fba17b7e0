// jbu_fast.cu -- joint bilateral upsampling (a6, Eq.2) fused with the
// reprojection (a7, Eq.3) and the valid-point count, sm_100a.
//
// Eq.2 with R-15..R-19, R-24: for full-res pixel p, taps q in the (2R+1)^2 window
// around c = floor(p/s):  D_p = s * sum_q w_q D'_q / sum_q w_q,
//   log2 w_q = sx[tx] + sy[ty] - cr * (dist2(I_p, I_q) - ref)
// with sx, sy = -log2(e)|p_down - q|^2/(2 sigma_s^2) split per axis (separable),
// cr = log2(e)/(2 sigma_r^2), dist2 = the exact integer squared RGB distance
// (VABSDIFF4 + IDP4A).  `ref` is any per-pixel constant (it cancels in the
// ratio); it is the centre tap's dist2 when cr*that <= 4 (one pass, exponents
// stay small so f32 rounding of the exponent is tiny), else the window minimum
// (an extra integer pass).  Out-of-image taps get sx or sy = -inf (weight 0),
// matching "taps outside the low-res image are skipped".  Rows are accumulated
// separately and scaled by 2^sy at the end of the row.
//
// k_jbu_fast (any s): one thread = one full-res pixel; block = 32 x 8 pixels; the block's low-res
// taps (guide sample + label) are staged once in shared memory as 8-byte records.
// The reprojection [X Y Z W] = Q [u v D_p 1] follows in registers; xyz is written
// through shared memory as coalesced 16-byte stores; one atomic per block counts
// the points with D_p >= min_disp.
#include <math.h>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

constexpr int JB_X = 32, JB_Y = 8, JB_RMAX = 8;
constexpr int JB_LW = JB_X + 2 * JB_RMAX + 1, JB_LH = JB_Y + 2 * JB_RMAX + 1;

struct JbuFastArgs {
    int W, H, s;
    float inv_s, cs, cr;
    float q[16];
    float min_disp;
    int do_xyz;
};

__device__ __forceinline__ float ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int R>
__global__ void __launch_bounds__(256) k_jbu_fast(const int32_t *__restrict__ disp_lo, const uint8_t *__restrict__ guide,
                                                  float *__restrict__ disp_hi, float *__restrict__ xyz,
                                                  unsigned long long *__restrict__ n_valid, JbuFastArgs a)
{
    __shared__ uint2 sT[JB_LW * JB_LH];
    __shared__ __align__(16) float sX[JB_Y][JB_X * 3];
    __shared__ unsigned warp_cnt[8];
    const int b = blockIdx.z;
    const int s = a.s;
    const int Wh = a.W * s, Hh = a.H * s;
    const int x0 = blockIdx.x * JB_X, y0 = blockIdx.y * JB_Y;
    const int lx0 = x0 / s - R, ly0 = y0 / s - R;
    const int lw = min(x0 + JB_X - 1, Wh - 1) / s + R - lx0 + 1;
    const int lh = min(y0 + JB_Y - 1, Hh - 1) / s + R - ly0 + 1;
    const uint8_t *G = guide + (size_t)b * Hh * Wh * 3;
    const int32_t *Dl = disp_lo + (size_t)b * a.H * a.W;
    const int tid = threadIdx.y * JB_X + threadIdx.x;
    for (int e = tid; e < lw * lh; e += JB_X * JB_Y) {
        const int qy = ly0 + e / lw, qx = lx0 + e % lw;
        uint2 rec = make_uint2(0u, 0u);
        if (qx >= 0 && qy >= 0 && qx < a.W && qy < a.H) {
            const uint8_t *g = G + ((size_t)(s * qy + s / 2) * Wh + (size_t)(s * qx + s / 2)) * 3;
            rec.x = (unsigned)g[0] | ((unsigned)g[1] << 8) | ((unsigned)g[2] << 16);
            rec.y = __float_as_uint((float)Dl[(size_t)qy * a.W + qx]);
        }
        sT[e] = rec;
    }
    __syncthreads();
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    const bool inside = x < Wh && y < Hh;
    float Dp = 0.f;
    if (inside) {
        const uint8_t *gp = G + ((size_t)y * Wh + x) * 3;
        const unsigned Ip = (unsigned)gp[0] | ((unsigned)gp[1] << 8) | ((unsigned)gp[2] << 16);
        const int cx = x / s, cy = y / s;
        const float fx = (x + 0.5f) * a.inv_s - 0.5f - (float)cx;  // p_down - c, in (-0.5, 0.5)
        const float fy = (y + 0.5f) * a.inv_s - 0.5f - (float)cy;
        float sxl[2 * R + 1], syl[2 * R + 1];
#pragma unroll
        for (int t = 0; t < 2 * R + 1; ++t) {
            const float dx = fx + (float)(R - t), dy = fy + (float)(R - t);
            const int qx = cx - R + t, qy = cy - R + t;
            sxl[t] = (qx >= 0 && qx < a.W) ? -a.cs * dx * dx : -INFINITY;
            syl[t] = (qy >= 0 && qy < a.H) ? -a.cs * dy * dy : -INFINITY;
        }
        const int e0 = (cy - R - ly0) * lw + (cx - R - lx0);
        const uint2 cen = sT[e0 + R * lw + R];
        unsigned ad = __vabsdiffu4(Ip, cen.x);
        int ref = (int)__dp4a(ad, ad, 0u);
        if (a.cr * (float)ref > 4.0f) {
            // the centre is far in colour: reference the window minimum instead
#pragma unroll
            for (int ty = 0; ty < 2 * R + 1; ++ty) {
                if (syl[ty] == -INFINITY) continue;
#pragma unroll
                for (int tx = 0; tx < 2 * R + 1; ++tx) {
                    if (sxl[tx] == -INFINITY) continue;
                    const unsigned adq = __vabsdiffu4(Ip, sT[e0 + ty * lw + tx].x);
                    ref = min(ref, (int)__dp4a(adq, adq, 0u));
                }
            }
        }
        // exact float of (dist2 - ref) via the 2^23 magic: |dist2 - ref| < 2^22
        const int off = (1 << 22) - ref;
        float num = 0.f, den = 0.f;
#pragma unroll
        for (int ty = 0; ty < 2 * R + 1; ++ty) {
            float nr = 0.f, dr = 0.f;
#pragma unroll
            for (int tx = 0; tx < 2 * R + 1; ++tx) {
                const uint2 t = sT[e0 + ty * lw + tx];
                const unsigned adq = __vabsdiffu4(Ip, t.x);
                const int n = (int)__dp4a(adq, adq, 0u) + off;
                const float f = __int_as_float(0x4B000000 | n) - 12582912.0f;  // = dist2 - ref
                const float w = ex2(fmaf(-a.cr, f, sxl[tx]));
                nr = fmaf(w, __uint_as_float(t.y), nr);
                dr += w;
            }
            const float rf = ex2(syl[ty]);
            num = fmaf(rf, nr, num);
            den = fmaf(rf, dr, den);
        }
        Dp = (float)s * (num / den);
        disp_hi[((size_t)b * Hh + y) * Wh + x] = Dp;
    }
    if (!a.do_xyz) return;
    // ---- a7: reprojection of this pixel, Eq.3 with Q (R-20, R-21)
    const bool valid = inside && Dp >= a.min_disp;
    float o0 = __int_as_float(0x7fc00000), o1 = o0, o2 = o0;
    if (valid) {
        const float fu = (float)x, fv = (float)y;
        const float X = fmaf(a.q[0], fu, fmaf(a.q[1], fv, fmaf(a.q[2], Dp, a.q[3])));
        const float Y = fmaf(a.q[4], fu, fmaf(a.q[5], fv, fmaf(a.q[6], Dp, a.q[7])));
        const float Z = fmaf(a.q[8], fu, fmaf(a.q[9], fv, fmaf(a.q[10], Dp, a.q[11])));
        const float Wq = fmaf(a.q[12], fu, fmaf(a.q[13], fv, fmaf(a.q[14], Dp, a.q[15])));
        o0 = X / Wq;
        o1 = Y / Wq;
        o2 = Z / Wq;
    }
    float *row = sX[threadIdx.y];
    row[3 * threadIdx.x] = o0;
    row[3 * threadIdx.x + 1] = o1;
    row[3 * threadIdx.x + 2] = o2;
    const unsigned m = __ballot_sync(FULL, valid);
    if (threadIdx.x == 0) warp_cnt[threadIdx.y] = __popc(m);
    __syncwarp();
    // the warp's 32 pixels are contiguous: 96 floats = 24 float4 when aligned
    if (y < Hh) {
        const int nx = min(JB_X, Wh - x0);
        float *dst = xyz + (((size_t)b * Hh + y) * Wh + x0) * 3;
        if (nx == JB_X && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
            if (threadIdx.x < 24)
                reinterpret_cast<float4 *>(dst)[threadIdx.x] = reinterpret_cast<const float4 *>(row)[threadIdx.x];
        } else {
            for (int k = threadIdx.x; k < 3 * nx; k += 32) dst[k] = row[k];
        }
    }
    __syncthreads();
    if (tid == 0) {
        unsigned n = 0;
#pragma unroll
        for (int w = 0; w < JB_Y; ++w) n += warp_cnt[w];
        if (n) atomicAdd(n_valid + b, (unsigned long long)n);
    }
}

// ---------------------------------------------------------------- P pixels per thread
// k_jbu_vec: same arithmetic as k_jbu_fast, bit for bit, for s % P == 0 (P = 2, 4).
// A thread owns P horizontally adjacent full-res pixels of one footprint row: they
// share the window centre c, so each tap record is read from shared memory once
// for P pixels, the row factor 2^sy is shared, and pixel pairs run on the packed
// FP32x2 datapath (FADD2/FFMA2).  The integer squared RGB distance comes out of
// IDP4A already as the float bit pattern 2^23 + (dist2 - ref): the accumulator
// input is 0x4B000000 + 2^22 - ref.  Per pixel-tap: VABSDIFF4, IDP4A, 1/2 FADD2,
// 1/2 FFMA2, MUFU.EX2, 1/2 FFMA2, 1/2 FADD2 -- the EX2 (16/clk/SM) is the bound.
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

template <int P> struct GuideVec;
template <> struct GuideVec<4> {  // 12 bytes, 4-byte aligned (x0 % 4 == 0)
    static __device__ __forceinline__ void load(const uint8_t *g, unsigned I[4])
    {
        const unsigned *w = reinterpret_cast<const unsigned *>(g);
        const unsigned w0 = __ldg(w), w1 = __ldg(w + 1), w2 = __ldg(w + 2);
        I[0] = w0 & 0xFFFFFFu;
        I[1] = __funnelshift_r(w0, w1, 24) & 0xFFFFFFu;
        I[2] = __funnelshift_r(w1, w2, 16) & 0xFFFFFFu;
        I[3] = w2 >> 8;
    }
};
template <> struct GuideVec<2> {  // 6 bytes, 2-byte aligned
    static __device__ __forceinline__ void load(const uint8_t *g, unsigned I[2])
    {
        const unsigned short *h = reinterpret_cast<const unsigned short *>(g);
        const unsigned h0 = __ldg(h), h1 = __ldg(h + 1), h2 = __ldg(h + 2);
        I[0] = h0 | ((h1 & 0xFFu) << 16);
        I[1] = (h1 >> 8) | (h2 << 8);
    }
};

template <int R, int P>
__global__ void __launch_bounds__(256) k_jbu_vec(const int32_t *__restrict__ disp_lo, const uint8_t *__restrict__ guide,
                                                 float *__restrict__ disp_hi, float *__restrict__ xyz,
                                                 unsigned long long *__restrict__ n_valid, JbuFastArgs a)
{
    constexpr int T = 2 * R + 1;
    __shared__ uint2 sT[JB_LW * JB_LH];
    __shared__ unsigned warp_cnt[8];
    const int b = blockIdx.z;
    const int s = a.s;
    const int Wh = a.W * s, Hh = a.H * s;
    const int x0 = blockIdx.x * (JB_X * P), y0 = blockIdx.y * JB_Y;
    const int lx0 = x0 / s - R, ly0 = y0 / s - R;
    const int lw = min(x0 + JB_X * P - 1, Wh - 1) / s + R - lx0 + 1;
    const int lh = min(y0 + JB_Y - 1, Hh - 1) / s + R - ly0 + 1;
    const uint8_t *G = guide + (size_t)b * Hh * Wh * 3;
    const int32_t *Dl = disp_lo + (size_t)b * a.H * a.W;
    const int tid = threadIdx.y * JB_X + threadIdx.x;
    for (int e = tid; e < lw * lh; e += JB_X * JB_Y) {
        const int qy = ly0 + e / lw, qx = lx0 + e % lw;
        uint2 rec = make_uint2(0u, 0u);
        if (qx >= 0 && qy >= 0 && qx < a.W && qy < a.H) {
            const uint8_t *g = G + ((size_t)(s * qy + s / 2) * Wh + (size_t)(s * qx + s / 2)) * 3;
            rec.x = (unsigned)g[0] | ((unsigned)g[1] << 8) | ((unsigned)g[2] << 16);
            rec.y = __float_as_uint((float)Dl[(size_t)qy * a.W + qx]);
        }
        sT[e] = rec;
    }
    __syncthreads();
    const int x = x0 + P * threadIdx.x, y = y0 + threadIdx.y;
    const bool inside = x < Wh && y < Hh;  // Wh % P == 0: all P pixels or none
    float Dp[P];
#pragma unroll
    for (int k = 0; k < P; ++k) Dp[k] = 0.f;
    if (inside) {
        unsigned Ip[P];
        GuideVec<P>::load(G + ((size_t)y * Wh + x) * 3, Ip);
        const int cx = x / s, cy = y / s;
        const float fy = (y + 0.5f) * a.inv_s - 0.5f - (float)cy;
        float syl[T];
        f2_t sx2[P / 2][T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const float dy = fy + (float)(R - t);
            const int qy = cy - R + t, qx = cx - R + t;
            syl[t] = (qy >= 0 && qy < a.H) ? -a.cs * dy * dy : -INFINITY;
            const bool okx = qx >= 0 && qx < a.W;
#pragma unroll
            for (int j = 0; j < P / 2; ++j) {
                const float fx0 = (x + 2 * j + 0.5f) * a.inv_s - 0.5f - (float)cx;
                const float fx1 = (x + 2 * j + 1.5f) * a.inv_s - 0.5f - (float)cx;
                const float d0 = fx0 + (float)(R - t), d1 = fx1 + (float)(R - t);
                sx2[j][t] = pk2(okx ? -a.cs * d0 * d0 : -INFINITY, okx ? -a.cs * d1 * d1 : -INFINITY);
            }
        }
        const int e0 = (cy - R - ly0) * lw + (cx - R - lx0);
        const unsigned cen = sT[e0 + R * lw + R].x;
        int ref[P];
        bool far = false;
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const unsigned ad = __vabsdiffu4(Ip[k], cen);
            ref[k] = (int)__dp4a(ad, ad, 0u);
            far = far || a.cr * (float)ref[k] > 4.0f;
        }
        if (far) {
            // some centre is far in colour: reference that pixel's window minimum
            float sxk[T];
#pragma unroll
            for (int t = 0; t < T; ++t) {
                float u, v;
                upk2(sx2[0][t], u, v);
                sxk[t] = u;
            }
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const unsigned ad = __vabsdiffu4(Ip[k], cen);
                if (!(a.cr * (float)__dp4a(ad, ad, 0u) > 4.0f)) continue;
                for (int ty = 0; ty < T; ++ty) {
                    if (syl[ty] == -INFINITY) continue;
                    for (int tx = 0; tx < T; ++tx) {
                        if (sxk[tx] == -INFINITY) continue;
                        const unsigned adq = __vabsdiffu4(Ip[k], sT[e0 + ty * lw + tx].x);
                        ref[k] = min(ref[k], (int)__dp4a(adq, adq, 0u));
                    }
                }
            }
        }
        unsigned acc[P];
#pragma unroll
        for (int k = 0; k < P; ++k) acc[k] = 0x4B000000u + (1u << 22) - (unsigned)ref[k];
        const f2_t magic = pk2(-12582912.0f, -12582912.0f);
        const f2_t ncr = pk2(-a.cr, -a.cr);
        f2_t num[P / 2], den[P / 2];
#pragma unroll
        for (int j = 0; j < P / 2; ++j) num[j] = den[j] = 0ull;
#pragma unroll
        for (int ty = 0; ty < T; ++ty) {
            f2_t nr[P / 2], dr[P / 2];
#pragma unroll
            for (int j = 0; j < P / 2; ++j) nr[j] = dr[j] = 0ull;
            const uint2 *row = sT + e0 + ty * lw;
#pragma unroll
            for (int tx = 0; tx < T; ++tx) {
                const uint2 tp = row[tx];
                const float dq = __uint_as_float(tp.y);
                const f2_t dd = pk2(dq, dq);
#pragma unroll
                for (int j = 0; j < P / 2; ++j) {
                    const unsigned a0 = __vabsdiffu4(Ip[2 * j], tp.x), a1 = __vabsdiffu4(Ip[2 * j + 1], tp.x);
                    const f2_t F = pk2(__uint_as_float(__dp4a(a0, a0, acc[2 * j])),
                                       __uint_as_float(__dp4a(a1, a1, acc[2 * j + 1])));
                    const f2_t ex = fma2(ncr, add2(F, magic), sx2[j][tx]);
                    float e0f, e1f;
                    upk2(ex, e0f, e1f);
                    const f2_t w = pk2(ex2(e0f), ex2(e1f));
                    nr[j] = fma2(w, dd, nr[j]);
                    dr[j] = add2(w, dr[j]);
                }
            }
            const float rf = ex2(syl[ty]);
            const f2_t rf2 = pk2(rf, rf);
#pragma unroll
            for (int j = 0; j < P / 2; ++j) {
                num[j] = fma2(rf2, nr[j], num[j]);
                den[j] = fma2(rf2, dr[j], den[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < P / 2; ++j) {
            float n0, n1, d0, d1;
            upk2(num[j], n0, n1);
            upk2(den[j], d0, d1);
            Dp[2 * j] = (float)s * (n0 / d0);
            Dp[2 * j + 1] = (float)s * (n1 / d1);
        }
        float *dst = disp_hi + ((size_t)b * Hh + y) * Wh + x;
        if (P == 4)
            *reinterpret_cast<float4 *>(dst) = make_float4(Dp[0], Dp[1], Dp[2], Dp[3]);
        else
            *reinterpret_cast<float2 *>(dst) = make_float2(Dp[0], Dp[1]);
    }
    if (!a.do_xyz) return;
    // ---- a7: reprojection, Eq.3 with Q (R-20, R-21); 3P contiguous floats per thread
    float o[3 * P];
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const bool valid = inside && Dp[k] >= a.min_disp;
        float o0 = __int_as_float(0x7fc00000), o1 = o0, o2 = o0;
        if (valid) {
            const float fu = (float)(x + k), fv = (float)y, D = Dp[k];
            const float X = fmaf(a.q[0], fu, fmaf(a.q[1], fv, fmaf(a.q[2], D, a.q[3])));
            const float Y = fmaf(a.q[4], fu, fmaf(a.q[5], fv, fmaf(a.q[6], D, a.q[7])));
            const float Z = fmaf(a.q[8], fu, fmaf(a.q[9], fv, fmaf(a.q[10], D, a.q[11])));
            const float Wq = fmaf(a.q[12], fu, fmaf(a.q[13], fv, fmaf(a.q[14], D, a.q[15])));
            o0 = X / Wq;
            o1 = Y / Wq;
            o2 = Z / Wq;
            ++cnt;
        }
        o[3 * k] = o0;
        o[3 * k + 1] = o1;
        o[3 * k + 2] = o2;
    }
    if (inside) {
        float *dst = xyz + (((size_t)b * Hh + y) * Wh + x) * 3;
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
    cnt = __reduce_add_sync(FULL, cnt);
    if (threadIdx.x == 0) warp_cnt[threadIdx.y] = (unsigned)cnt;
    __syncthreads();
    if (tid == 0) {
        unsigned n = 0;
#pragma unroll
        for (int w = 0; w < JB_Y; ++w) n += warp_cnt[w];
        if (n) atomicAdd(n_valid + b, (unsigned long long)n);
    }
}

template <int P>
static void launch_vec(int radius, dim3 grid, dim3 block, cudaStream_t st, const int32_t *disp_lo,
                       const uint8_t *guide, float *disp_hi, float *xyz, unsigned long long *n_valid,
                       const JbuFastArgs &a)
{
    switch (radius) {
    case 1: k_jbu_vec<1, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    case 2: k_jbu_vec<2, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    case 3: k_jbu_vec<3, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    case 4: k_jbu_vec<4, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    case 5: k_jbu_vec<5, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    case 6: k_jbu_vec<6, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    case 7: k_jbu_vec<7, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    default: k_jbu_vec<8, P><<<grid, block, 0, st>>>(disp_lo, guide, disp_hi, xyz, n_valid, a); break;
    }
}

cudaError_t launch_jbu_fast(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide, int s, float *disp_hi,
                            float sigma_s, float sigma_r, int radius, const float *Qf, float min_disp, float *xyz,
                            unsigned long long *n_valid, cudaStream_t st)
{
    const double log2e = 1.4426950408889634;
    JbuFastArgs a;
    a.W = W;
    a.H = H;
    a.s = s;
    a.inv_s = (float)(1.0 / s);
    a.cs = (float)(log2e / (2.0 * (double)sigma_s * sigma_s));
    a.cr = (float)(log2e / (2.0 * (double)sigma_r * sigma_r));
    for (int i = 0; i < 16; ++i) a.q[i] = Qf ? Qf[i] : 0.f;
    a.min_disp = min_disp;
    a.do_xyz = xyz != nullptr;
    dim3 block(JB_X, JB_Y);
    // the vector path needs P-aligned guide words and 4P-byte aligned outputs
    const auto al = [](const void *p, uintptr_t m) { return ((uintptr_t)p & (m - 1)) == 0; };
    int P = (s % 4 == 0) ? 4 : (s % 2 == 0) ? 2 : 1;
    if (P == 4 && !(al(guide, 4) && al(disp_hi, 16) && al(xyz, 16))) P = (al(guide, 2) && al(disp_hi, 8) && al(xyz, 8)) ? 2 : 1;
    if (P == 2 && !(al(guide, 2) && al(disp_hi, 8) && al(xyz, 8))) P = 1;
    if (P > 1) {
        dim3 grid((W * s + JB_X * P - 1) / (JB_X * P), (H * s + JB_Y - 1) / JB_Y, B);
        if (P == 4)
            launch_vec<4>(radius, grid, block, st, disp_lo, guide, disp_hi, xyz, n_valid, a);
        else
            launch_vec<2>(radius, grid, block, st, disp_lo, guide, disp_hi, xyz, n_valid, a);
        note_launch();
        return cudaGetLastError();
    }
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
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
