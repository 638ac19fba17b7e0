// Microbenchmark: integer ALU throughput on this GPU (lane-ops / clock / SM) of the
// instructions the message update is built from -- each in 8 independent chains per
// thread, 64 warps per SM.  Guides the u16x2 formulation in bp_fast.cu.
#include <cstdio>
#include <cuda_runtime.h>

// 8 INDEPENDENT chains per thread (each chain only feeds itself) so that the rate
// measured is the pipe's throughput, not a dependency chain's latency
#define BODY(EXPR)                                                                 \
    unsigned v[8];                                                                 \
    for (int c = 0; c < 8; ++c) v[c] = seed * (threadIdx.x + 3 * c);               \
    const unsigned s = seed | 0x00800080u, t = 0x7F007F00u ^ seed, u = seed * 7u;   \
    for (int i = 0; i < iters; ++i) {                                              \
        _Pragma("unroll") for (int c = 0; c < 8; ++c) {                            \
            const unsigned a = v[c];                                               \
            v[c] = (EXPR);                                                         \
        }                                                                          \
    }                                                                              \
    unsigned r = 0;                                                                \
    for (int c = 0; c < 8; ++c) r ^= v[c];                                         \
    if (r == 0x12345u) out[0] = r;

__global__ void k_viaddmin(unsigned *out, int iters, unsigned seed) { BODY(__viaddmin_u16x2(a, s, t)) }
__global__ void k_viaddmin_s(unsigned *out, int iters, unsigned seed) { BODY((unsigned)__viaddmin_s16x2(a, s, t)) }
__global__ void k_vmin(unsigned *out, int iters, unsigned seed) { BODY(__vminu2(a, t) + s) }
__global__ void k_vmin3(unsigned *out, int iters, unsigned seed) { BODY(__vimin3_u16x2(a, t, u) + s) }
__global__ void k_imin(unsigned *out, int iters, unsigned seed) { BODY(min(a, t) + s) }
__global__ void k_iadd3(unsigned *out, int iters, unsigned seed) { BODY(a + s + (a >> 3)) }
__global__ void k_prmt(unsigned *out, int iters, unsigned seed)
{
    BODY(__byte_perm(a, s, 0x6240) + t)
}

typedef void (*kfn)(unsigned *, int, unsigned);

int main()
{
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    unsigned *out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 8192, threads = 256, blocks = sms * 8;
    const struct { const char *name; kfn f; } ks[] = {
        {"VIADDMNMX.U16x2 (__viaddmin_u16x2)", k_viaddmin}, {"VIADDMNMX.S16x2 (__viaddmin_s16x2)", k_viaddmin_s},
        {"VIMNMX.U16x2 (__vminu2) [+IADD]", k_vmin}, {"VIMNMX3.U16x2 (__vimin3_u16x2) [+IADD]", k_vmin3},
        {"IMNMX (32-bit min) [+IADD]", k_imin}, {"IADD3 [+SHF]", k_iadd3}, {"PRMT [+IADD]", k_prmt}};
    for (auto &k : ks) {
        float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k.f<<<blocks, threads>>>(out, iters, 12345u);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        const double ops = (double)blocks * threads * iters * 8;
        printf("%-40s %6.1f instr-lanes/clk/SM\n", k.name, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    return 0;
}
