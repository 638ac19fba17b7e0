// csbp.cu -- row f2: constant-space belief propagation (the paper's [4]),
// sm_100a.  Definition: DESIGN.md R-32..R-35 (oracle/vsbp_oracle.c oracle_csbp).
//
// Level l keeps k_l = min(L, k0 2^l) candidate labels per pixel; memory per pixel is
// O(k_l) instead of O(L): candidates (u16), their data costs (i32) and the four
// incoming messages (i32, receiver-stored, over the receiver's candidates).
//   * k_csbp_top: one CTA per top-level pixel computes D_T(p, d) for every label
//     from the images (footprint sums over 2^T x 2^T full-resolution pixels, read
//     through L1) and keeps the k_T least (ties: smaller label) by ranking;
//   * k_csbp_init: one thread per pixel of a finer level scores the parent's
//     candidates (D_l + the parent's four incoming messages), keeps the k_l least
//     and inherits the parent's messages for them;
//   * k_csbp_update: one checkerboard colour; a thread per pixel computes its
//     four outgoing messages over each neighbour's candidates (O(k^2)), min-
//     normalised, and writes them into the neighbour's incoming slots (the
//     neighbours are the other colour, so there is no race);
//   * k_csbp_wta: label of least D + sum of incoming at level 0.
// The data term of a candidate is evaluated directly from the grey images --
// the cost volume is never materialised ("constant space").
#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

// data cost of label d summed over the footprint [x0,x1) x [y0,y1) (R-2, R-8)
__device__ __forceinline__ int footprint_cost(const uint8_t *lb, const uint8_t *rb, int W, int x0, int x1, int y0,
                                              int y1, int d, int lam_q, int tau_d)
{
    int s = 0;
    for (int y = y0; y < y1; ++y)
        for (int x = x0; x < x1; ++x)
            s += (x - d >= 0) ? lam_q * min(abs((int)__ldg(lb + (size_t)y * W + x) - (int)__ldg(rb + (size_t)y * W + x - d)),
                                            tau_d)
                              : lam_q * tau_d;
    return s;
}

// ---------------------------------------------------------------- top level
constexpr int CT_T = 256, CT_LMAX = 512;

__global__ void __launch_bounds__(CT_T) k_csbp_top(const uint8_t *__restrict__ left, const uint8_t *__restrict__ right,
                                                   CsbpArgs a, CsbpLevel lv)
{
    __shared__ int sD[CT_LMAX];
    __shared__ unsigned char sSel[CT_LMAX];
    const int b = blockIdx.y, p = blockIdx.x;
    const int X = p % lv.W, Y = p / lv.W;
    const int f = 1 << lv.l;
    const int x0 = X * f, x1 = min(x0 + f, a.W), y0 = Y * f, y1 = min(y0 + f, a.H);
    const uint8_t *lb = left + (size_t)b * a.W * a.H, *rb = right + (size_t)b * a.W * a.H;
    for (int d = threadIdx.x; d < a.L; d += CT_T) sD[d] = footprint_cost(lb, rb, a.W, x0, x1, y0, y1, d, a.lam_q, a.tau_d);
    __syncthreads();
    for (int d = threadIdx.x; d < a.L; d += CT_T) {
        const int v = sD[d];
        int rank = 0;
        for (int e = 0; e < a.L; ++e) rank += (sD[e] < v || (sD[e] == v && e < d)) ? 1 : 0;
        sSel[d] = rank < lv.k ? 1 : 0;
    }
    __syncthreads();
    const size_t base = ((size_t)b * lv.n + p) * lv.k;
    for (int d = threadIdx.x; d < a.L; d += CT_T) {
        if (!sSel[d]) continue;
        int pos = 0;
        for (int e = 0; e < d; ++e) pos += sSel[e];
        lv.cand[base + pos] = (uint16_t)d;
        lv.dsel[base + pos] = sD[d];
    }
    for (int e = threadIdx.x; e < 4 * lv.k; e += CT_T) lv.msg[base * 4 + e] = 0;
}

// ---------------------------------------------------------------- finer levels
__global__ void __launch_bounds__(128) k_csbp_init(const uint8_t *__restrict__ left, const uint8_t *__restrict__ right,
                                                   CsbpArgs a, CsbpLevel lv, CsbpLevel pv)
{
    const int b = blockIdx.y;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= lv.n) return;
    const int X = p % lv.W, Y = p / lv.W;
    const int P = (Y >> 1) * pv.W + (X >> 1);
    const int f = 1 << lv.l;
    const int x0 = X * f, x1 = min(x0 + f, a.W), y0 = Y * f, y1 = min(y0 + f, a.H);
    const uint8_t *lb = left + (size_t)b * a.W * a.H, *rb = right + (size_t)b * a.W * a.H;
    const size_t pb = ((size_t)b * pv.n + P) * pv.k;
    const int kp = pv.k;
    int D[CS_KMAX];
    long long sc[CS_KMAX];
    for (int i = 0; i < kp; ++i) {
        const int d = pv.cand[pb + i];
        D[i] = footprint_cost(lb, rb, a.W, x0, x1, y0, y1, d, a.lam_q, a.tau_d);
        long long s = D[i];
        for (int q = 0; q < 4; ++q) s += pv.msg[pb * 4 + (size_t)q * kp + i];
        sc[i] = s;
    }
    const bool has[4] = {Y > 0, Y < lv.H - 1, X > 0, X < lv.W - 1};
    const size_t base = ((size_t)b * lv.n + p) * lv.k;
    int pos = 0;
    for (int i = 0; i < kp; ++i) {
        int rank = 0;
        for (int j = 0; j < kp; ++j) rank += (sc[j] < sc[i] || (sc[j] == sc[i] && j < i)) ? 1 : 0;
        if (rank >= lv.k) continue;
        lv.cand[base + pos] = pv.cand[pb + i];
        lv.dsel[base + pos] = D[i];
        for (int q = 0; q < 4; ++q) lv.msg[base * 4 + (size_t)q * lv.k + pos] = has[q] ? pv.msg[pb * 4 + (size_t)q * kp + i] : 0;
        ++pos;
    }
}

// ---------------------------------------------------------------- message update
template <int KM>
__global__ void __launch_bounds__(128) k_csbp_update(CsbpArgs a, CsbpLevel lv, int colour)
{
    const int b = blockIdx.y;
    const int Wc = (lv.W + 1) >> 1;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= Wc * lv.H) return;
    const int y = t / Wc, x = 2 * (t - y * Wc) + ((y + colour) & 1);
    if (x >= lv.W) return;
    const int k = lv.k;
    const size_t p = (size_t)b * lv.n + (size_t)y * lv.W + x;
    int cp[KM], D[KM], in[4][KM];
#pragma unroll
    for (int i = 0; i < KM; ++i) {
        if (i < k) {
            cp[i] = lv.cand[p * k + i];
            D[i] = lv.dsel[p * k + i];
#pragma unroll
            for (int q = 0; q < 4; ++q) in[q][i] = lv.msg[p * 4 * k + (size_t)q * k + i];
        }
    }
    const bool has[4] = {y > 0, y < lv.H - 1, x > 0, x < lv.W - 1};
    const int dxs[4] = {0, 0, -1, 1}, dys[4] = {-1, 1, 0, 0}, opp[4] = {1, 0, 3, 2};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        if (!has[kk]) continue;
        const size_t q = (size_t)b * lv.n + (size_t)(y + dys[kk]) * lv.W + (x + dxs[kk]);
        int h[KM];
        int hmin = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < KM; ++i) {
            if (i < k) {
                int s = D[i];
#pragma unroll
                for (int q2 = 0; q2 < 4; ++q2)
                    if (q2 != kk && has[q2]) s += in[q2][i];
                h[i] = s;
                hmin = min(hmin, s);
            }
        }
        int m[KM];
        int mmin = 0x7fffffff;
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            if (j < k) {
                const int cq = lv.cand[q * k + j];
                int best = hmin + a.tau_q;
#pragma unroll
                for (int i = 0; i < KM; ++i)
                    if (i < k) best = min(best, h[i] + a.S * abs(cp[i] - cq));
                m[j] = best;
                mmin = min(mmin, best);
            }
        }
        int *dst = lv.msg + q * 4 * k + (size_t)opp[kk] * k;
#pragma unroll
        for (int j = 0; j < KM; ++j)
            if (j < k) dst[j] = m[j] - mmin;
    }
}

template <int KM>
__global__ void __launch_bounds__(128) k_csbp_wta(CsbpLevel lv, int32_t *__restrict__ disp)
{
    const int b = blockIdx.y;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= lv.n) return;
    const int k = lv.k;
    const size_t base = (size_t)b * lv.n + p;
    int best = 0x7fffffff, lab = 0;
#pragma unroll
    for (int i = 0; i < KM; ++i) {
        if (i < k) {
            int s = lv.dsel[base * k + i];
#pragma unroll
            for (int q = 0; q < 4; ++q) s += lv.msg[base * 4 * k + (size_t)q * k + i];
            if (s < best) {  // candidates ascend: the first minimum is the smaller label
                best = s;
                lab = lv.cand[base * k + i];
            }
        }
    }
    disp[base] = lab;
}

// ---------------------------------------------------------------- parallel variants
// k_csbp_top_rows: the top level's data term with the footprint staged in shared
// memory and one (label, footprint row) pair per thread, reduced with shared
// atomics (integer: order-independent).
__global__ void __launch_bounds__(CT_T) k_csbp_top_rows(const uint8_t *__restrict__ left,
                                                        const uint8_t *__restrict__ right, CsbpArgs a, CsbpLevel lv)
{
    extern __shared__ __align__(16) unsigned char tsm[];
    __shared__ int sD[CT_LMAX];
    __shared__ unsigned char sSel[CT_LMAX];
    const int b = blockIdx.y, p = blockIdx.x;
    const int X = p % lv.W, Y = p / lv.W;
    const int f = 1 << lv.l;
    const int x0 = X * f, x1 = min(x0 + f, a.W), y0 = Y * f, y1 = min(y0 + f, a.H);
    const int fw = x1 - x0, fh = y1 - y0, span = fw + a.L - 1;
    uint8_t *sl = tsm;              // [fh][fw]
    uint8_t *sr = tsm + f * f;      // [fh][span]: right columns x0-L+1 .. x1-1
    const uint8_t *lb = left + (size_t)b * a.W * a.H, *rb = right + (size_t)b * a.W * a.H;
    for (int e = threadIdx.x; e < fw * fh; e += CT_T)
        sl[e] = __ldg(lb + (size_t)(y0 + e / fw) * a.W + x0 + e % fw);
    for (int e = threadIdx.x; e < span * fh; e += CT_T) {
        const int r = e / span, j = e - r * span, x = x0 - a.L + 1 + j;
        sr[e] = x >= 0 ? __ldg(rb + (size_t)(y0 + r) * a.W + x) : 0;
    }
    for (int d = threadIdx.x; d < a.L; d += CT_T) sD[d] = 0;
    __syncthreads();
    const int border = a.lam_q * a.tau_d;
    for (int e = threadIdx.x; e < a.L * fh; e += CT_T) {
        const int d = e % a.L, r = e / a.L;
        int s = 0;
        for (int i = 0; i < fw; ++i) {
            const int x = x0 + i;
            s += (x - d >= 0) ? a.lam_q * min(abs((int)sl[r * fw + i] - (int)sr[r * span + i + a.L - 1 - d]), a.tau_d)
                              : border;
        }
        atomicAdd(&sD[d], s);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < a.L; d += CT_T) {
        const int v = sD[d];
        int rank = 0;
        for (int e = 0; e < a.L; ++e) rank += (sD[e] < v || (sD[e] == v && e < d)) ? 1 : 0;
        sSel[d] = rank < lv.k ? 1 : 0;
    }
    __syncthreads();
    const size_t base = ((size_t)b * lv.n + p) * lv.k;
    for (int d = threadIdx.x; d < a.L; d += CT_T) {
        if (!sSel[d]) continue;
        int pos = 0;
        for (int e = 0; e < d; ++e) pos += sSel[e];
        lv.cand[base + pos] = (uint16_t)d;
        lv.dsel[base + pos] = sD[d];
    }
    for (int e = threadIdx.x; e < 4 * lv.k; e += CT_T) lv.msg[base * 4 + e] = 0;
}

// k_csbp_init_par: one thread per (pixel, parent candidate); GP = pow2 >= k_{l+1}
// lanes per pixel, CTA of 128 threads; ranks from shared memory.
__global__ void __launch_bounds__(128) k_csbp_init_par(const uint8_t *__restrict__ left,
                                                       const uint8_t *__restrict__ right, CsbpArgs a, CsbpLevel lv,
                                                       CsbpLevel pv, int GP)
{
    __shared__ long long ssc[128];
    __shared__ unsigned char ssel[128];
    const int b = blockIdx.y;
    const int lane = threadIdx.x % GP, grp = threadIdx.x / GP;
    const int p = blockIdx.x * (128 / GP) + grp;
    const int kp = pv.k;
    const bool act = p < lv.n && lane < kp;
    int X = 0, Y = 0, Dv = 0, lab = 0;
    size_t pb = 0;
    long long sc = 0x7fffffffffffffffll;
    if (act) {
        X = p % lv.W;
        Y = p / lv.W;
        const int P = (Y >> 1) * pv.W + (X >> 1);
        const int f = 1 << lv.l;
        const int x0 = X * f, x1 = min(x0 + f, a.W), y0 = Y * f, y1 = min(y0 + f, a.H);
        pb = ((size_t)b * pv.n + P) * kp;
        lab = pv.cand[pb + lane];
        Dv = footprint_cost(left + (size_t)b * a.W * a.H, right + (size_t)b * a.W * a.H, a.W, x0, x1, y0, y1, lab,
                            a.lam_q, a.tau_d);
        sc = Dv;
        for (int q = 0; q < 4; ++q) sc += pv.msg[pb * 4 + (size_t)q * kp + lane];
    }
    ssc[threadIdx.x] = sc;
    __syncthreads();
    int rank = 0;
    const int g0 = grp * GP;
    for (int j = 0; j < kp; ++j) {
        const long long o = ssc[g0 + j];
        rank += (o < sc || (o == sc && j < lane)) ? 1 : 0;
    }
    const bool keep = act && rank < lv.k;
    ssel[threadIdx.x] = keep ? 1 : 0;
    __syncthreads();
    if (!keep) return;
    int pos = 0;
    for (int j = 0; j < lane; ++j) pos += ssel[g0 + j];
    const size_t base = ((size_t)b * lv.n + p) * lv.k;
    const bool has[4] = {Y > 0, Y < lv.H - 1, X > 0, X < lv.W - 1};
    lv.cand[base + pos] = (uint16_t)lab;
    lv.dsel[base + pos] = Dv;
    for (int q = 0; q < 4; ++q) lv.msg[base * 4 + (size_t)q * lv.k + pos] = has[q] ? pv.msg[pb * 4 + (size_t)q * kp + lane] : 0;
}

// k_csbp_update_par: one thread per (sender pixel, receiver candidate j); GP = pow2 >= k
// lanes per pixel (up to 64: the minimum over two warps goes through shared memory);
// the sender's h is rebuilt per lane from L1-resident rows.  The serial k_csbp_update
// (one thread per pixel, O(k^2) in a thread) was 368 us per launch on C4's 43 x 24
// top level at k = 64 (ncu, r02): too few threads.
__global__ void __launch_bounds__(128) k_csbp_update_par(CsbpArgs a, CsbpLevel lv, int colour, int GP)
{
    const int b = blockIdx.y;
    const int Wc = (lv.W + 1) >> 1;
    const int lane = threadIdx.x % GP;
    const int t = blockIdx.x * (128 / GP) + threadIdx.x / GP;
    const int k = lv.k;
    bool act = t < Wc * lv.H;
    int x = 0, y = 0;
    if (act) {
        y = t / Wc;
        x = 2 * (t - y * Wc) + ((y + colour) & 1);
        act = x < lv.W;
    }
    const bool lj = act && lane < k;
    const size_t p = (size_t)b * lv.n + (size_t)y * lv.W + x;
    const bool has[4] = {y > 0, y < lv.H - 1, x > 0, x < lv.W - 1};
    const int dxs[4] = {0, 0, -1, 1}, dys[4] = {-1, 1, 0, 0}, opp[4] = {1, 0, 3, 2};
    const uint16_t *cp = lv.cand + p * k;
    const int32_t *Dp = lv.dsel + p * k, *inp = lv.msg + p * 4 * k;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        const bool go = lj && has[kk];
        int m = 0x7fffffff;
        if (go) {
            const size_t q = (size_t)b * lv.n + (size_t)(y + dys[kk]) * lv.W + (x + dxs[kk]);
            const int cq = lv.cand[q * k + lane];
            int hmin = 0x7fffffff, best = 0x7fffffff;
            for (int i = 0; i < k; ++i) {
                int h = Dp[i];
#pragma unroll
                for (int q2 = 0; q2 < 4; ++q2)
                    if (q2 != kk) h += inp[q2 * k + i];
                hmin = min(hmin, h);
                best = min(best, h + a.S * abs((int)cp[i] - cq));
            }
            m = min(best, hmin + a.tau_q);
        }
        int mmin = m;
        for (int o = min(GP, 32) >> 1; o > 0; o >>= 1) mmin = min(mmin, __shfl_xor_sync(0xffffffffu, mmin, o, min(GP, 32)));
        if (GP > 32) {  // GP = 64: the pixel's two warps combine their minima (block-uniform branch)
            __shared__ int wmin[4];
            if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = mmin;
            __syncthreads();
            mmin = min(wmin[threadIdx.x >> 5], wmin[(threadIdx.x >> 5) ^ 1]);
            __syncthreads();
        }
        if (go) {
            const size_t q = (size_t)b * lv.n + (size_t)(y + dys[kk]) * lv.W + (x + dxs[kk]);
            lv.msg[q * 4 * k + (size_t)opp[kk] * k + lane] = m - mmin;
        }
    }
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_csbp_top(const uint8_t *left, const uint8_t *right, const CsbpArgs &a, const CsbpLevel &lv, int B,
                            cudaStream_t st)
{
    if (a.L > CT_LMAX) return cudaErrorInvalidValue;
    const int f = 1 << lv.l;
    const size_t smem = (size_t)f * f + (size_t)f * (f + a.L - 1);
    if (smem <= 40 * 1024)
        k_csbp_top_rows<<<dim3(lv.n, B), CT_T, smem, st>>>(left, right, a, lv);
    else
        k_csbp_top<<<dim3(lv.n, B), CT_T, 0, st>>>(left, right, a, lv);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_csbp_init(const uint8_t *left, const uint8_t *right, const CsbpArgs &a, const CsbpLevel &lv,
                             const CsbpLevel &pv, int B, cudaStream_t st)
{
    if (pv.k > CS_KMAX) return cudaErrorInvalidValue;
    int GP = 1;
    while (GP < pv.k) GP <<= 1;
    if (GP >= 4) {
        const int ppb = 128 / GP;
        k_csbp_init_par<<<dim3((lv.n + ppb - 1) / ppb, B), 128, 0, st>>>(left, right, a, lv, pv, GP);
    } else {
        k_csbp_init<<<dim3((lv.n + 127) / 128, B), 128, 0, st>>>(left, right, a, lv, pv);
    }
    note_launch();
    return cudaGetLastError();
}

#define VSBP_CS_K(KERNEL, ARGS)                      \
    if (lv.k <= 1) KERNEL<1><<<grid, 128, 0, st>>> ARGS;        \
    else if (lv.k <= 2) KERNEL<2><<<grid, 128, 0, st>>> ARGS;   \
    else if (lv.k <= 4) KERNEL<4><<<grid, 128, 0, st>>> ARGS;   \
    else if (lv.k <= 8) KERNEL<8><<<grid, 128, 0, st>>> ARGS;   \
    else if (lv.k <= 16) KERNEL<16><<<grid, 128, 0, st>>> ARGS; \
    else if (lv.k <= 32) KERNEL<32><<<grid, 128, 0, st>>> ARGS; \
    else KERNEL<64><<<grid, 128, 0, st>>> ARGS;

cudaError_t launch_csbp_update(const CsbpArgs &a, const CsbpLevel &lv, int colour, int B, cudaStream_t st)
{
    if (lv.k > CS_KMAX) return cudaErrorInvalidValue;
    const int nc = ((lv.W + 1) >> 1) * lv.H;
    if (lv.k >= 8) {  // GP = pow2 >= k lanes per pixel (k = 33..64: two warps per pixel)
        int GP = 1;
        while (GP < lv.k) GP <<= 1;
        const int ppb = 128 / GP;
        k_csbp_update_par<<<dim3((nc + ppb - 1) / ppb, B), 128, 0, st>>>(a, lv, colour, GP);
        note_launch();
        return cudaGetLastError();
    }
    const dim3 grid((nc + 127) / 128, B);
    VSBP_CS_K(k_csbp_update, (a, lv, colour))
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_csbp_wta(const CsbpLevel &lv, int32_t *disp, int B, cudaStream_t st)
{
    if (lv.k > CS_KMAX) return cudaErrorInvalidValue;
    const dim3 grid((lv.n + 127) / 128, B);
    VSBP_CS_K(k_csbp_wta, (lv, disp))
    note_launch();
    return cudaGetLastError();
}
#undef VSBP_CS_K

}  // namespace vsbp

namespace vsbp {
__global__ void k_u16_to_i32(const uint16_t *__restrict__ in, int32_t *__restrict__ out, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

cudaError_t launch_csbp_export(const uint16_t *cand, size_t n, int32_t *out, cudaStream_t st)
{
    k_u16_to_i32<<<(unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, st>>>(cand, out, n);
    note_launch();
    return cudaGetLastError();
}
}  // namespace vsbp
