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
// One thread = one full-res pixel; block = 32 x 8 pixels; the block's low-res
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
    dim3 grid((W * s + JB_X - 1) / JB_X, (H * s + JB_Y - 1) / JB_Y, B);
    dim3 block(JB_X, JB_Y);
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
