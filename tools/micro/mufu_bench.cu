// Microbenchmark: MUFU.EX2 throughput on this GPU (ops / clock / SM), alone and
// mixed with the JBU inner loop's other instructions.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x)
{
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int CH>
__global__ void k_ex2(float *out, int iters, float seed)
{
    float v[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = seed * (threadIdx.x + c) * 1e-6f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) v[c] = ex2(v[c]) - 1.0f;
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += v[c];
    if (s == 12345.f) out[0] = s;
}

// the JBU per pixel-tap mix: VABSDIFF4 + IDP4A + FADD + FFMA + EX2 + FFMA + FADD
template <int CH>
__global__ void k_mix(float *out, int iters, unsigned seed)
{
    unsigned ip[CH];
    float num[CH], den[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        ip[c] = seed * (threadIdx.x + 7 * c);
        num[c] = den[c] = 0.f;
    }
    unsigned t = seed ^ threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        t = t * 1664525u + 1013904223u;
        const float dq = (float)(t & 63);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const unsigned ad = __vabsdiffu4(ip[c], t);
            const float f = __uint_as_float(__dp4a(ad, ad, 0x4B000000u)) - 8388608.0f;
            const float w = ex2(fmaf(-0.0032f, f, -0.5f));
            num[c] = fmaf(w, dq, num[c]);
            den[c] += w;
        }
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += num[c] / den[c];
    if (s == 12345.f) out[0] = s;
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz (max)
    float *out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int warps = 8; warps <= 32; warps *= 2) {
        const int threads = 256, blocks = sms * warps * 32 / threads;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_ex2<8><<<blocks, threads>>>(out, iters, 1.0f);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double ops = (double)blocks * threads * iters * 8;
            if (rep) printf("ex2 alone   warps/SM=%2d: %.2f ops/clk/SM (at %d MHz max clock)\n", warps,
                            ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
            cudaEventRecord(a);
            k_mix<8><<<blocks, threads>>>(out, iters, 12345u);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("jbu mix     warps/SM=%2d: %.2f pixel-taps/clk/SM\n", warps,
                            ops / (ms * 1e-3) / sms / (clk * 1e3));
        }
    }
    return 0;
}
