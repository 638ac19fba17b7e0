// pipeline_kernels.cu -- rows a0, a6, a7, a8 of the hot path on sm_100a.
//
//   k_prep       a0  RGB -> grey (77R+150G+29B+128)>>8 -> s x s mean, half up  P:26, R-22
//   k_jbu        a6  joint bilateral upsampling, Eq.2, f32                      P:34-38, R-15..R-19, R-24
//   k_reproject  a7  [X Y Z W]^T = Q [u v d 1]^T, NaN below min_disp          P:40-44 Eq.3, R-20, R-21
//   k_summary    a8  label sum + order-independent label hash per pair
#include <math.h>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

// ======================================================================== a0
__global__ void __launch_bounds__(256) k_prep(const uint8_t *__restrict__ rgb, int W_hi, int H_hi, int s, int n,
                                              uint8_t *__restrict__ gray)
{
    const int W = W_hi / s, H = H_hi / s;
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long)n * W * H) return;
    const int f = (int)(t / ((long)W * H));
    const long r = t - (long)f * W * H;
    const int Y = (int)(r / W), X = (int)(r - (long)Y * W);
    const uint8_t *base = rgb + (size_t)f * H_hi * W_hi * 3;
    int sum = 0;
    for (int j = 0; j < s; ++j) {
        const uint8_t *row = base + ((size_t)(Y * s + j) * W_hi + (size_t)X * s) * 3;
        for (int i = 0; i < s; ++i) {
            const int R = row[3 * i], G = row[3 * i + 1], Bc = row[3 * i + 2];
            sum += (77 * R + 150 * G + 29 * Bc + 128) >> 8;
        }
    }
    const int n2 = s * s;
    gray[t] = (uint8_t)((sum + n2 / 2) / n2);
}

// ======================================================================== a6
// Block = 32 x 8 full-res pixels of one pair.  The low-res taps it can touch
// (window centres floor(x/s) +- r) are staged once in shared memory: the guide
// sample I_q packed as u8x4 and the label D'_q.
constexpr int JBU_BX = 32, JBU_BY = 8, JBU_RMAX = 8;
constexpr int JBU_LW = JBU_BX + 2 * JBU_RMAX, JBU_LH = JBU_BY + 2 * JBU_RMAX;

struct JbuArgs {
    int W, H, s, r;
    float inv_s;
    float cs;  // log2(e) / (2 sigma_s^2), sigma_s in low-res px
    float cr;  // log2(e) / (2 sigma_r^2)
};

__global__ void __launch_bounds__(256) k_jbu(const int32_t *__restrict__ disp_lo, const uint8_t *__restrict__ guide,
                                             float *__restrict__ disp_hi, JbuArgs a)
{
    __shared__ unsigned sI[JBU_LW * JBU_LH];
    __shared__ int sD[JBU_LW * JBU_LH];
    const int b = blockIdx.z;
    const int Wh = a.W * a.s, Hh = a.H * a.s;
    const int x0 = blockIdx.x * JBU_BX, y0 = blockIdx.y * JBU_BY;
    const int lx0 = x0 / a.s - a.r, ly0 = y0 / a.s - a.r;
    const int lw = min(x0 + JBU_BX - 1, Wh - 1) / a.s + a.r - lx0 + 1;
    const int lh = min(y0 + JBU_BY - 1, Hh - 1) / a.s + a.r - ly0 + 1;
    const uint8_t *G = guide + (size_t)b * Hh * Wh * 3;
    const int32_t *Dl = disp_lo + (size_t)b * a.H * a.W;
    const int tid = threadIdx.y * JBU_BX + threadIdx.x;
    for (int e = tid; e < lw * lh; e += JBU_BX * JBU_BY) {
        const int qy = ly0 + e / lw, qx = lx0 + e % lw;
        unsigned I = 0;
        int dv = -1;  // -1: outside the low-res image, skipped
        if (qx >= 0 && qy >= 0 && qx < a.W && qy < a.H) {
            const uint8_t *g = G + ((size_t)(a.s * qy + a.s / 2) * Wh + (size_t)(a.s * qx + a.s / 2)) * 3;
            I = (unsigned)g[0] | ((unsigned)g[1] << 8) | ((unsigned)g[2] << 16);
            dv = Dl[(size_t)qy * a.W + qx];
        }
        sI[e] = I;
        sD[e] = dv;
    }
    __syncthreads();
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    if (x >= Wh || y >= Hh) return;
    const uint8_t *gp = G + ((size_t)y * Wh + x) * 3;
    const unsigned Ip = (unsigned)gp[0] | ((unsigned)gp[1] << 8) | ((unsigned)gp[2] << 16);
    const float px = (x + 0.5f) * a.inv_s - 0.5f, py = (y + 0.5f) * a.inv_s - 0.5f;
    const int cx = x / a.s, cy = y / a.s;
    const int e0 = (cy - a.r - ly0) * lw + (cx - a.r - lx0);
    const int n = 2 * a.r + 1;
    // pass 1: the smallest squared colour distance (exact integer)
    int dmin = 0x7fffffff;
    for (int ty = 0; ty < n; ++ty)
        for (int tx = 0; tx < n; ++tx) {
            const int e = e0 + ty * lw + tx;
            if (sD[e] < 0) continue;
            const unsigned ad = __vabsdiffu4(Ip, sI[e]);
            dmin = min(dmin, (int)__dp4a(ad, ad, 0u));
        }
    // pass 2: the largest logit, logit = -cs |p_down - q|^2 - cr (dist2 - dmin)  (log2 units)
    float lmax = -INFINITY;
    for (int ty = 0; ty < n; ++ty)
        for (int tx = 0; tx < n; ++tx) {
            const int e = e0 + ty * lw + tx;
            if (sD[e] < 0) continue;
            const unsigned ad = __vabsdiffu4(Ip, sI[e]);
            const float sx = px - (float)(cx - a.r + tx), sy = py - (float)(cy - a.r + ty);
            const float l = -a.cs * (sx * sx + sy * sy) - a.cr * (float)((int)__dp4a(ad, ad, 0u) - dmin);
            lmax = fmaxf(lmax, l);
        }
    // pass 3: Eq.2 with w = 2^(logit - max), accumulated relative to the centre label
    const int dc = sD[e0 + a.r * lw + a.r];
    float num = 0.f, den = 0.f;
    for (int ty = 0; ty < n; ++ty)
        for (int tx = 0; tx < n; ++tx) {
            const int e = e0 + ty * lw + tx;
            const int dq = sD[e];
            if (dq < 0) continue;
            const unsigned ad = __vabsdiffu4(Ip, sI[e]);
            const float sx = px - (float)(cx - a.r + tx), sy = py - (float)(cy - a.r + ty);
            const float l = -a.cs * (sx * sx + sy * sy) - a.cr * (float)((int)__dp4a(ad, ad, 0u) - dmin);
            const float w = exp2f(l - lmax);
            num = fmaf(w, (float)(dq - dc), num);
            den += w;
        }
    disp_hi[((size_t)b * Hh + y) * Wh + x] = (float)a.s * ((float)dc + num / den);
}

// ======================================================================== a7
struct QMat {
    float q[16];
};

__global__ void __launch_bounds__(256) k_reproject(const float *__restrict__ disp, int W, int H, QMat Q,
                                                   float min_disp, float *__restrict__ xyz,
                                                   unsigned long long *__restrict__ n_valid)
{
    const int b = blockIdx.y;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const bool inb = idx < W * H;
    bool valid = false;
    if (inb) {
        const int v = idx / W, u = idx - v * W;
        const float d = disp[(size_t)b * W * H + idx];
        valid = d >= min_disp;
        float o0 = __int_as_float(0x7fc00000), o1 = o0, o2 = o0;
        if (valid) {
            const float fu = (float)u, fv = (float)v;
            const float X = fmaf(Q.q[0], fu, fmaf(Q.q[1], fv, fmaf(Q.q[2], d, Q.q[3])));
            const float Y = fmaf(Q.q[4], fu, fmaf(Q.q[5], fv, fmaf(Q.q[6], d, Q.q[7])));
            const float Z = fmaf(Q.q[8], fu, fmaf(Q.q[9], fv, fmaf(Q.q[10], d, Q.q[11])));
            const float Wq = fmaf(Q.q[12], fu, fmaf(Q.q[13], fv, fmaf(Q.q[14], d, Q.q[15])));
            o0 = X / Wq;
            o1 = Y / Wq;
            o2 = Z / Wq;
        }
        float *o = xyz + ((size_t)b * W * H + idx) * 3;
        o[0] = o0;
        o[1] = o1;
        o[2] = o2;
    }
    // one atomic per block: warp ballots -> shared-memory sum
    __shared__ unsigned warp_cnt[8];
    const unsigned m = __ballot_sync(FULL, valid);
    if ((threadIdx.x & 31) == 0) warp_cnt[threadIdx.x >> 5] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned n = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) n += warp_cnt[w];
        if (n) atomicAdd(n_valid + b, (unsigned long long)n);
    }
}

// ======================================================================== a8
__device__ __forceinline__ unsigned long long mix64(unsigned long long z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct Summary {
    unsigned long long n_valid;
    long long label_sum;
    unsigned long long label_hash;
    unsigned long long pair_id;
    unsigned long long reserved[4];
};

__global__ void k_summary_init(int B, const unsigned long long *__restrict__ n_valid, unsigned long long first,
                               Summary *__restrict__ out)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    Summary s = {};
    s.n_valid = n_valid ? n_valid[b] : 0ull;
    s.pair_id = first + b;
    out[b] = s;
}

__global__ void __launch_bounds__(256) k_summary(const int32_t *__restrict__ disp, int N, Summary *__restrict__ out)
{
    const int b = blockIdx.y;
    long long sum = 0;
    unsigned long long hash = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const int d = disp[(size_t)b * N + i];
        sum += d;
        hash += mix64(((unsigned long long)i << 32) | (unsigned)d);
    }
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(FULL, sum, o);
        hash += __shfl_xor_sync(FULL, hash, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&out[b].label_sum), (unsigned long long)sum);
        atomicAdd(&out[b].label_hash, hash);
    }
}

// ======================================================================== launchers
cudaError_t launch_prep(int n, const uint8_t *rgb, int W_hi, int H_hi, int s, uint8_t *gray, cudaStream_t st)
{
    const long threads = (long)n * (W_hi / s) * (H_hi / s);
    k_prep<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(rgb, W_hi, H_hi, s, n, gray);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_jbu(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide, int s, float *disp_hi,
                       float sigma_s, float sigma_r, int radius, cudaStream_t st)
{
    const double log2e = 1.4426950408889634;
    JbuArgs a;
    a.W = W;
    a.H = H;
    a.s = s;
    a.r = radius;
    a.inv_s = (float)(1.0 / s);
    a.cs = (float)(log2e / (2.0 * (double)sigma_s * sigma_s));
    a.cr = (float)(log2e / (2.0 * (double)sigma_r * sigma_r));
    dim3 grid((W * s + JBU_BX - 1) / JBU_BX, (H * s + JBU_BY - 1) / JBU_BY, B);
    k_jbu<<<grid, dim3(JBU_BX, JBU_BY), 0, st>>>(disp_lo, guide, disp_hi, a);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_reproject(int B, const float *disp, int W, int H, const float Qf[16], float min_disp, float *xyz,
                             unsigned long long *n_valid, cudaStream_t st)
{
    QMat Q;
    for (int i = 0; i < 16; ++i) Q.q[i] = Qf[i];
    dim3 grid((W * H + 255) / 256, B);
    k_reproject<<<grid, 256, 0, st>>>(disp, W, H, Q, min_disp, xyz, n_valid);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_summary(int B, const int32_t *disp, int W, int H, const unsigned long long *n_valid,
                           uint64_t first_pair_id, void *summary, cudaStream_t st)
{
    Summary *out = (Summary *)summary;
    k_summary_init<<<(B + 127) / 128, 128, 0, st>>>(B, n_valid, first_pair_id, out);
    const int N = W * H;
    dim3 grid(min((N + 255) / 256, 64), B);
    k_summary<<<grid, 256, 0, st>>>(disp, N, out);
    note_launch(2);
    return cudaGetLastError();
}

}  // namespace vsbp
