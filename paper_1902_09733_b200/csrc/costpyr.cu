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
#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

constexpr int CP_T = 16;  // level-0 tile side (levels 0..4 of a tile nest inside it)

__device__ __forceinline__ void store_chunk(void *base, int bytes, size_t off, const int v[CH])
{
    if (bytes == 1)
        Chunk<uint8_t>::store((uint8_t *)base + off, v);
    else if (bytes == 2)
        Chunk<uint16_t>::store((uint16_t *)base + off, v);
    else
        Chunk<int32_t>::store((int32_t *)base + off, v);
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
                store_chunk(a.D[0], a.dbytes[0],
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

    // ---- levels 2..F-1 (a2) from the previous level in shared memory
    int *prev = sD;
    int Tp = TQ;
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

size_t costpyr_smem(int L, int Lp, int F)
{
    const size_t img = (size_t)CP_T * CP_T + (size_t)CP_T * (CP_T + L - 1);
    size_t px = 0;  // levels 1..F-2 are staged (the last fused level is only written)
    for (int l = 1, T = CP_T / 2; l < F - 1; ++l, T >>= 1) px += (size_t)T * T;
    return ((img + 15) & ~(size_t)15) + px * Lp * sizeof(int);
}

cudaError_t launch_costpyr(const uint8_t *left, const uint8_t *right, CostPyrArgs a, int B, cudaStream_t st)
{
    const size_t img = (size_t)CP_T * CP_T + (size_t)CP_T * (CP_T + a.L - 1);
    a.img_smem = (int)((img + 15) & ~(size_t)15);
    const size_t smem = costpyr_smem(a.L, a.Lp, a.F);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_costpyr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((a.W[0] + CP_T - 1) / CP_T, (a.H[0] + CP_T - 1) / CP_T, B);
    k_costpyr<<<grid, 256, smem, st>>>(left, right, a);
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
