// rectify.cu -- row f1: radial undistortion + bilinear remap fused with row a0
// (grey + s x s box mean), sm_100a.
//
// P:26 (§2.1): radial distortion only, "rectify and undistort individual images
// ... cvInitUndistortMap() and cvRemap()"; R-26, R-27.
// For destination pixel (u,v) of an n-frame batch:
//   x = (u-c_u)/f_u, y = (v-c_v)/f_v, r2 = x*x + y*y,
//   kr = 1 + k1 r2 + k2 r2 r2 + k3 r2 r2 r2, src = (f_u x kr + c_u, f_v y kr + c_v)
// in IEEE double, left to right, no contraction (explicit _rn intrinsics), then
// quantised to 1/32 px: q = floor(32 src + 0.5), i = floor(q/32), a = q - 32 i.
// Each channel is (sum wx_i wy_j I(i+., j+.) + 512) >> 10 with wx = {32-ax, ax},
// wy = {32-ay, ay}, taps outside the image reading 0; the rectified RGB feeds the
// BT.601 grey and the box mean of row a0 exactly as k_prep computes them.
//
// Cvremap's table is not materialised: the map of a destination pixel is
// recomputed in FP64 (B200 runs FP64 at ~1/2 the FP32 rate), once per launch and
// reused for all n frames of the batch -- reading a 33 MB map per frame would cost
// more HBM time than the frame itself.  One thread = one low-res output pixel; per
// footprint row it computes the s source coordinates, then for every frame
// gathers the 2x2 taps (two 8-byte loads per tap row), writes the rectified row
// (optional) and accumulates the grey sum.
#include <math.h>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

constexpr int RP_MAXF = 16;    // frames per launch (the host loops above this)

struct RectArgs {
    int W, H, s, n;            // full-res frame, footprint, frames
    int aligned;               // frames start on 8-byte boundaries: 8-byte tap loads
    double fu, fv, cu, cv, k1, k2, k3;
};

// source coordinate of destination pixel (u, v) in 1/32 px (R-26)
__device__ __forceinline__ void undistort_q(const RectArgs &a, int u, int v, int &qx, int &qy)
{
    const double x = __ddiv_rn(__dsub_rn((double)u, a.cu), a.fu);
    const double y = __ddiv_rn(__dsub_rn((double)v, a.cv), a.fv);
    const double r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    double kr = __dadd_rn(1.0, __dmul_rn(a.k1, r2));
    kr = __dadd_rn(kr, __dmul_rn(__dmul_rn(a.k2, r2), r2));
    kr = __dadd_rn(kr, __dmul_rn(__dmul_rn(__dmul_rn(a.k3, r2), r2), r2));
    const double su = __dadd_rn(__dmul_rn(__dmul_rn(a.fu, x), kr), a.cu);
    const double sv = __dadd_rn(__dmul_rn(__dmul_rn(a.fv, y), kr), a.cv);
    qx = (int)floor(__dadd_rn(__dmul_rn(su, 32.0), 0.5));
    qy = (int)floor(__dadd_rn(__dmul_rn(sv, 32.0), 0.5));
}

// bytes [off, off+6) of the 16 bytes lo|hi (little endian): two RGB taps
__device__ __forceinline__ unsigned long long take6(unsigned long long lo, unsigned long long hi, int off)
{
    return off == 0 ? lo : (lo >> (8 * off)) | (hi << (64 - 8 * off));
}

template <int s>
__global__ void __launch_bounds__(256) k_rectify_prep(const uint8_t *__restrict__ raw, uint8_t *__restrict__ gray,
                                                      uint8_t *__restrict__ rect, RectArgs a)
{
    const int W = a.W, H = a.H;
    const int Wl = W / s, Hl = H / s;
    __shared__ unsigned ssum[RP_MAXF][256];  // per-thread grey sums, one per frame
    __shared__ int sq[2][s][256];             // this footprint row's source coordinates
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= Wl * Hl) return;
    const int Y = t / Wl, X = t - Y * Wl;
    const size_t frame = (size_t)W * H * 3;
    for (int f = 0; f < a.n; ++f) ssum[f][threadIdx.x] = 0u;
    for (int jy = 0; jy < s; ++jy) {
        const int v = Y * s + jy;
#pragma unroll 1
        for (int jx = 0; jx < s; ++jx) undistort_q(a, X * s + jx, v, sq[0][jx][threadIdx.x], sq[1][jx][threadIdx.x]);
#pragma unroll 1
        for (int f = 0; f < a.n; ++f) {
            const uint8_t *img = raw + (size_t)f * frame;
            unsigned rowsum = 0u;
#pragma unroll 1
            for (int jx = 0; jx < s; ++jx) {
                const int qx = sq[0][jx][threadIdx.x], qy = sq[1][jx][threadIdx.x];
                const int ix = qx >> 5, iy = qy >> 5;  // arithmetic shift = floor
                const int ax = qx & 31, ay = qy & 31;
                const int wx0 = 32 - ax, wy0 = 32 - ay;
                int acc[3] = {0, 0, 0};
                const size_t b0 = 3 * ((size_t)iy * W + ix);
                const bool fast =
                    a.aligned && ix >= 0 && iy >= 0 && ix + 1 < W && iy + 1 < H && b0 + 3 * (size_t)W + 16 <= frame;
                if (fast) {
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const size_t base = b0 + (size_t)j * 3 * W;
                        const uint2 *p = reinterpret_cast<const uint2 *>(img + (base & ~(size_t)7));
                        const uint2 w0 = __ldg(p), w1 = __ldg(p + 1);
                        const unsigned long long lo = ((unsigned long long)w0.y << 32) | w0.x;
                        const unsigned long long hi = ((unsigned long long)w1.y << 32) | w1.x;
                        const unsigned long long px = take6(lo, hi, (int)(base & 7));
                        const int wy = j ? ay : wy0;
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            const int t0 = (int)((px >> (8 * c)) & 0xff), t1 = (int)((px >> (8 * (c + 3))) & 0xff);
                            acc[c] += wy * (wx0 * t0 + ax * t1);
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int py = iy + j, wy = j ? ay : wy0;
                        if (py < 0 || py >= H) continue;
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            const int pxx = ix + i, wx = i ? ax : wx0;
                            if (pxx < 0 || pxx >= W) continue;
                            const uint8_t *q = img + 3 * ((size_t)py * W + pxx);
#pragma unroll
                            for (int c = 0; c < 3; ++c) acc[c] += wy * wx * (int)q[c];
                        }
                    }
                }
                const int R = (acc[0] + 512) >> 10, G = (acc[1] + 512) >> 10, Bc = (acc[2] + 512) >> 10;
                if (rect) {
                    uint8_t *o = rect + (size_t)f * frame + 3 * ((size_t)v * W + X * s + jx);
                    o[0] = (uint8_t)R;
                    o[1] = (uint8_t)G;
                    o[2] = (uint8_t)Bc;
                }
                rowsum += (unsigned)((77 * R + 150 * G + 29 * Bc + 128) >> 8);
            }
            ssum[f][threadIdx.x] += rowsum;
        }
    }
    const unsigned n2 = (unsigned)(s * s);
    for (int f = 0; f < a.n; ++f) gray[(size_t)f * Wl * Hl + t] = (uint8_t)((ssum[f][threadIdx.x] + n2 / 2) / n2);
}

// the domain rule of R-26, identical to the oracle's
bool rectify_domain_ok(int W, int H, const double *cam)
{
    const double fu = cam[0], fv = cam[1], cu = cam[2], cv = cam[3];
    const double k1 = cam[4], k2 = cam[5], k3 = cam[6];
    const double xm = fmax(fabs((0.0 - cu) / fu), fabs(((double)(W - 1) - cu) / fu));
    const double ym = fmax(fabs((0.0 - cv) / fv), fabs(((double)(H - 1) - cv) / fv));
    const double r2m = xm * xm + ym * ym;
    const double K = 1.0 + fabs(k1) * r2m + fabs(k2) * r2m * r2m + fabs(k3) * r2m * r2m * r2m;
    return fu * xm * K + fabs(cu) < 16777216.0 && fv * ym * K + fabs(cv) < 16777216.0;
}

cudaError_t launch_rectify_prep(int n, const uint8_t *raw, int W, int H, const double *cam, int s, uint8_t *gray,
                                uint8_t *rect, cudaStream_t st)
{
    RectArgs a;
    a.W = W;
    a.H = H;
    a.s = s;
    a.fu = cam[0];
    a.fv = cam[1];
    a.cu = cam[2];
    a.cv = cam[3];
    a.k1 = cam[4];
    a.k2 = cam[5];
    a.k3 = cam[6];
    const int nl = (W / s) * (H / s);
    const size_t frame = (size_t)W * H * 3;
    a.aligned = ((uintptr_t)raw & 7) == 0 && frame % 8 == 0;
    for (int f0 = 0; f0 < n; f0 += RP_MAXF) {
        a.n = n - f0 < RP_MAXF ? n - f0 : RP_MAXF;
        const uint8_t *r = raw + (size_t)f0 * frame;
        uint8_t *g = gray + (size_t)f0 * nl, *o = rect ? rect + (size_t)f0 * frame : nullptr;
        const unsigned nb = (unsigned)((nl + 255) / 256);
        switch (s) {
        case 1: k_rectify_prep<1><<<nb, 256, 0, st>>>(r, g, o, a); break;
        case 2: k_rectify_prep<2><<<nb, 256, 0, st>>>(r, g, o, a); break;
        case 3: k_rectify_prep<3><<<nb, 256, 0, st>>>(r, g, o, a); break;
        case 4: k_rectify_prep<4><<<nb, 256, 0, st>>>(r, g, o, a); break;
        case 5: k_rectify_prep<5><<<nb, 256, 0, st>>>(r, g, o, a); break;
        case 6: k_rectify_prep<6><<<nb, 256, 0, st>>>(r, g, o, a); break;
        case 7: k_rectify_prep<7><<<nb, 256, 0, st>>>(r, g, o, a); break;
        default: k_rectify_prep<8><<<nb, 256, 0, st>>>(r, g, o, a); break;
        }
        note_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace vsbp
