// pipeline_kernels.cu -- rows a0, a7, a8 of the hot path on sm_100a (a6: jbu_fast.cu).
//
//   k_prep       a0  RGB -> grey (77R+150G+29B+128)>>8 -> s x s mean, half up  P:26, R-22
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

// s % 4 == 0: each footprint row is 3s/4 aligned 32-bit words (W_hi % 4 == 0 and the
// frame size is a multiple of 4), read as words; a warp's 32 pixels read
// contiguous 12s-byte runs per row.  Same arithmetic as k_prep.
template <int S4>
__global__ void __launch_bounds__(256) k_prep_w(const uint8_t *__restrict__ rgb, int W_hi, int H_hi, int n,
                                                uint8_t *__restrict__ gray)
{
    constexpr int s = 4 * S4, NW = 3 * S4;  // words per footprint row
    const int W = W_hi / s, H = H_hi / s;
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long)n * W * H) return;
    const int f = (int)(t / ((long)W * H));
    const long r = t - (long)f * W * H;
    const int Y = (int)(r / W), X = (int)(r - (long)Y * W);
    const uint8_t *base = rgb + (size_t)f * H_hi * W_hi * 3;
    int sum = 0;
#pragma unroll
    for (int j = 0; j < s; ++j) {
        const unsigned *row = reinterpret_cast<const unsigned *>(base + ((size_t)(Y * s + j) * W_hi + (size_t)X * s) * 3);
        unsigned w[NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) w[q] = __ldg(row + q);
#pragma unroll
        for (int i = 0; i < s; ++i) {
            const int R = (w[(3 * i) >> 2] >> (8 * ((3 * i) & 3))) & 0xff;
            const int G = (w[(3 * i + 1) >> 2] >> (8 * ((3 * i + 1) & 3))) & 0xff;
            const int Bc = (w[(3 * i + 2) >> 2] >> (8 * ((3 * i + 2) & 3))) & 0xff;
            sum += (77 * R + 150 * G + 29 * Bc + 128) >> 8;
        }
    }
    gray[t] = (uint8_t)((sum + s * s / 2) / (s * s));
}

// s == 4 with 16-byte aligned footprint rows (W_hi % 16 == 0, 16-byte aligned
// frames): a thread makes 4 adjacent output pixels of one row from 3 x 16-byte loads
// per footprint row (12 loads in flight per thread) and stores them as one word.
// Same arithmetic as k_prep.
__device__ __forceinline__ int grey_px(uint32_t w0, uint32_t w1, uint32_t w2, int k)
{
    // pixel k (0..3) of the 12 bytes w0 w1 w2: bytes 3k, 3k+1, 3k+2
    const uint32_t lo = k == 0 ? w0 : k == 1 ? __funnelshift_r(w0, w1, 24) : k == 2 ? __funnelshift_r(w1, w2, 16) : w2 >> 8;
    const int R = lo & 0xff, G = (lo >> 8) & 0xff, Bc = (lo >> 16) & 0xff;
    return (77 * R + 150 * G + 29 * Bc + 128) >> 8;
}

__global__ void __launch_bounds__(256) k_prep_v4(const uint8_t *__restrict__ rgb, int W_hi, int H_hi, int n,
                                                 uint8_t *__restrict__ gray)
{
    const int W = W_hi / 4, H = H_hi / 4, Wq = W / 4;
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long)n * Wq * H) return;
    const int f = (int)(t / ((long)Wq * H));
    const long r = t - (long)f * Wq * H;
    const int Y = (int)(r / Wq), xq = (int)(r - (long)Y * Wq);
    const uint8_t *base = rgb + (size_t)f * H_hi * W_hi * 3 + (size_t)xq * 48;
    uint4 v[4][3];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint4 *row = reinterpret_cast<const uint4 *>(base + (size_t)(Y * 4 + j) * W_hi * 3);
#pragma unroll
        for (int q = 0; q < 3; ++q) v[j][q] = __ldg(row + q);
    }
    uint32_t out = 0;
#pragma unroll
    for (int o = 0; o < 4; ++o) {  // output pixel o: input pixels 4o .. 4o+3 of each row (bytes 12o .. 12o+11)
        int sum = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t w[12] = {v[j][0].x, v[j][0].y, v[j][0].z, v[j][0].w, v[j][1].x, v[j][1].y,
                                    v[j][1].z, v[j][1].w, v[j][2].x, v[j][2].y, v[j][2].z, v[j][2].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) sum += grey_px(w[3 * o], w[3 * o + 1], w[3 * o + 2], k);
        }
        out |= (uint32_t)((sum + 8) / 16) << (8 * o);
    }
    *reinterpret_cast<uint32_t *>(gray + ((size_t)f * H + Y) * W + (size_t)xq * 4) = out;
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
    const int32_t *src = disp + (size_t)b * N;
    const int t0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    int i0 = 0;
    if ((N & 3) == 0 && ((uintptr_t)src & 15) == 0) {
        // four labels per 16-byte load (order-independent sums: same result)
        const int4 *s4 = reinterpret_cast<const int4 *>(src);
        for (int q = t0; q < N / 4; q += stride) {
            const int4 v = __ldg(s4 + q);
            const int d[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                sum += d[k];
                hash += mix64(((unsigned long long)(4 * q + k) << 32) | (unsigned)d[k]);
            }
        }
        i0 = N;
    }
    for (int i = i0 + t0; i < N; i += stride) {
        const int d = src[i];
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
    const unsigned nb = (unsigned)((threads + 255) / 256);
    if (s == 4 && W_hi % 16 == 0 && ((uintptr_t)rgb & 15) == 0 && ((uintptr_t)gray & 3) == 0) {
        const long tq = (long)n * (W_hi / 16) * (H_hi / 4);
        k_prep_v4<<<(unsigned)((tq + 255) / 256), 256, 0, st>>>(rgb, W_hi, H_hi, n, gray);
    } else if (s == 4 && ((uintptr_t)rgb & 3) == 0)
        k_prep_w<1><<<nb, 256, 0, st>>>(rgb, W_hi, H_hi, n, gray);
    else if (s == 8 && ((uintptr_t)rgb & 3) == 0)
        k_prep_w<2><<<nb, 256, 0, st>>>(rgb, W_hi, H_hi, n, gray);
    else
        k_prep<<<nb, 256, 0, st>>>(rgb, W_hi, H_hi, s, n, gray);
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
