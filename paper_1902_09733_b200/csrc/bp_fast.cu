// bp_fast.cu -- the packed message-update kernel (row a4, the hot loop), sm_100a.
//
// Same operation as k_update (bp_kernels.cu): one checkerboard colour of min-sum
// messages (Eq.1; R-9..R-12), bit-exact, but specialised for the common
// parameter domain (checked on the host, vsbp_api.cu):
//   * u8 message storage (tau_q <= 255) and S = 128, so tau_q <= 2S and the
//     truncated-linear lower envelope is an exact 3-tap stencil:
//       m(d) = min(h'(d), h'(d-1) + S, h'(d+1) + S),  h' = min(h - min h, tau_q)
//     (terms |d-d'| >= 2 cost >= 2S >= tau_q; clamping h' at tau_q does not change
//     min(., tau_q), and every stencil term is <= h'(d) <= tau_q);
//   * every belief of the level fits 16 bits (D_max + 4*tau_q < 2^16), so two
//     labels travel in one 32-bit register as u16x2 and the arithmetic runs on
//     the DPX 16x2 integer datapath (VIMNMX/VIMNMX3/VIADDMNMX .U16x2, plain IADD
//     on non-negative packed halves, PRMT for the u8 <-> u16x2 conversion).
// Register j of a thread's 16-label chunk holds (label d0+j, label d0+j+8); the
// storage order of vsbp_internal.cuh makes that a single PRMT per register.
// Neighbouring labels across chunks come from the adjacent lanes (2 shuffles per
// pair of directions); min_d h reduces over the G lanes (log2 G shuffles, two
// directions per shuffle).  HBM traffic per updated pixel: L*w_D + 8L bytes.
//
// WTA (a5) is fused into the last iteration of level 0 for the colour being
// updated there (its belief D + sum of 4 incoming is already in registers).
#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel)
{
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

// 16 u8 labels in storage order -> r[j] = (label j | label j+8 << 16)
__device__ __forceinline__ void unpack_u8(const uint4 w, uint32_t r[8])
{
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        r[2 * q] = prmt(u[q], 0u, 0x4240);      // bytes 0, 2 -> (2q, 2q+8)
        r[2 * q + 1] = prmt(u[q], 0u, 0x4341);  // bytes 1, 3 -> (2q+1, 2q+9)
    }
}

__device__ __forceinline__ uint4 pack_u8(const uint32_t r[8])
{
    uint32_t u[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) u[q] = prmt(r[2 * q], r[2 * q + 1], 0x6240);
    return make_uint4(u[0], u[1], u[2], u[3]);
}

template <typename TD> struct DLoad;
template <> struct DLoad<uint8_t> {
    static __device__ __forceinline__ void load(const uint8_t *p, uint32_t r[8])
    {
        unpack_u8(__ldg(reinterpret_cast<const uint4 *>(p)), r);
    }
};
template <> struct DLoad<uint16_t> {
    static __device__ __forceinline__ void load(const uint16_t *p, uint32_t r[8])
    {
        const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p));
        const uint4 b = __ldg(reinterpret_cast<const uint4 *>(p) + 1);
        r[0] = a.x, r[1] = a.y, r[2] = a.z, r[3] = a.w;
        r[4] = b.x, r[5] = b.y, r[6] = b.z, r[7] = b.w;
    }
};

// MODE 0: normal iteration; 1: top level t=0 (all incoming 0); 2: lower level t=0
// (incoming read from the parent level).  PAD: some labels of the chunk are >= L.
// WTA: also write the WTA label of the updated pixels to disp.
template <typename TD, int MODE, bool PAD, bool WTA>
__global__ void __launch_bounds__(256) k_update_fast(const TD *__restrict__ D, uint8_t *__restrict__ M,
                                                     const uint8_t *__restrict__ Mp, Geom g, int colour,
                                                     uint32_t SS, uint32_t TT, int32_t *__restrict__ disp)
{
    const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane_g = threadIdx.x & (g.G - 1);
    const long pix = gt >> g.log2G;
    const long per_c = (long)g.H * g.Wc;
    bool active = pix < (long)g.B * per_c;
    if (__all_sync(FULL, !active)) return;
    int b = 0, y = 0, i = 0, x = 0;
    if (active) {
        b = (int)(pix / per_c);
        const long r = pix - (long)b * per_c;
        y = (int)(r / g.Wc);
        i = (int)(r - (long)y * g.Wc);
        x = 2 * i + ((colour + y) & 1);
        active = x < g.W;
    }
    const bool io = active && lane_g < g.nch;
    const int d0 = lane_g * CH;
    const bool has[4] = {y > 0, y < g.H - 1, x > 0, x < g.W - 1};

    // ---- loads: the 4 incoming messages (neighbour q sends toward p on slot k^1), D
    uint4 wi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        wi[k] = make_uint4(0u, 0u, 0u, 0u);
        if (MODE == 1 || !io || !has[k]) continue;
        const int qx = x + (k == 2 ? -1 : (k == 3 ? 1 : 0));
        const int qy = y + (k == 0 ? -1 : (k == 1 ? 1 : 0));
        const uint8_t *src;
        if (MODE == 2) {
            const int px = qx >> 1, py = qy >> 1;
            src = Mp + m_off(b, (px + py) & 1, k ^ 1, py, px >> 1, g.Hp, g.Wcp, g.Lp) + d0;
        } else {
            src = M + m_off(b, colour ^ 1, k ^ 1, qy, qx >> 1, g.H, g.Wc, g.Lp) + d0;
        }
        wi[k] = __ldg(reinterpret_cast<const uint4 *>(src));
    }
    uint32_t tot[8];
    if (io) {
        DLoad<TD>::load(D + d_off(b, colour, y, i, g.H, g.Wc, g.Lp) + d0, tot);
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) tot[j] = 0u;
    }
    uint32_t in[4][8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        unpack_u8(wi[k], in[k]);
#pragma unroll
        for (int j = 0; j < 8; ++j) tot[j] += in[k][j];  // halves < 2^16: no carry
    }
    // labels >= L: 0xFFFF halves (excluded from min h, become tau_q after the clamp)
    uint32_t padm[8];
    if (PAD) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            padm[j] = (d0 + j >= g.L ? 0x0000FFFFu : 0u) | (d0 + j + 8 >= g.L ? 0xFFFF0000u : 0u);
    }

    // ---- fused WTA (a5): argmin of the belief tot, ties -> smallest d (R-13)
    if (WTA) {
        uint32_t best = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t lo = tot[j] & 0xFFFFu, hi = tot[j] >> 16;
            if (!PAD || d0 + j < g.L) best = min(best, (lo << 9) | (uint32_t)(d0 + j));
            if (!PAD || d0 + j + 8 < g.L) best = min(best, (hi << 9) | (uint32_t)(d0 + j + 8));
        }
        for (int o = g.G >> 1; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(FULL, best, o, g.G));
        if (active && lane_g == 0) disp[((size_t)b * g.H + y) * g.W + x] = (int32_t)(best & 511u);
    }

    // ---- the four outgoing messages, two directions at a time
#pragma unroll
    for (int kp = 0; kp < 4; kp += 2) {
        uint32_t h[2][8];
        uint32_t mn[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                h[e][j] = tot[j] - in[kp + e][j];
                if (PAD) h[e][j] |= padm[j];
            }
            const uint32_t a = __vimin3_u16x2(h[e][0], h[e][1], h[e][2]);
            const uint32_t c = __vimin3_u16x2(h[e][3], h[e][4], h[e][5]);
            const uint32_t d = __vimin3_u16x2(a, c, __vminu2(h[e][6], h[e][7]));
            mn[e] = __vminu2(d, prmt(d, 0u, 0x1032));  // min of both halves, in both halves
        }
        // min over the G lanes of the pixel: direction kp in the low half, kp+1 in the high half
        uint32_t pm = prmt(mn[0], mn[1], 0x5410);
        for (int o = g.G >> 1; o > 0; o >>= 1) pm = __vminu2(pm, __shfl_xor_sync(FULL, pm, o, g.G));
        const uint32_t hm[2] = {prmt(pm, 0u, 0x1010), prmt(pm, 0u, 0x3232)};
        // h' = min(h - min h, tau_q)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int j = 0; j < 8; ++j) h[e][j] = __vminu2(h[e][j] - hm[e], TT);
        // labels d0-1 (from lane-1: its r7 high half) and d0+16 (from lane+1: its r0 low half)
        uint32_t up = __shfl_up_sync(FULL, prmt(h[0][7], h[1][7], 0x7632), 1, g.G);
        uint32_t dn = __shfl_down_sync(FULL, prmt(h[0][0], h[1][0], 0x5410), 1, g.G);
        if (lane_g == 0) up = TT;
        if (lane_g == g.G - 1) dn = TT;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int k = kp + e;
            const uint32_t prev0 = prmt(up, h[e][7], e == 0 ? 0x5410 : 0x5432);  // (d0-1, d0+7)
            const uint32_t next7 = prmt(h[e][0], dn, e == 0 ? 0x5432 : 0x7632);  // (d0+8, d0+16)
            uint32_t o[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t pv = j == 0 ? prev0 : h[e][j - 1];
                const uint32_t nx = j == 7 ? next7 : h[e][j + 1];
                o[j] = __viaddmin_u16x2(pv, SS, __viaddmin_u16x2(nx, SS, h[e][j]));
                if (PAD) o[j] &= ~padm[j];
                if (!has[k]) o[j] = 0u;
            }
            if (io) *reinterpret_cast<uint4 *>(M + m_off(b, colour, k, y, i, g.H, g.Wc, g.Lp) + d0) = pack_u8(o);
        }
    }
}

cudaError_t launch_update_fast(const void *D, int dbytes, void *M, const void *Mp, const Geom &g, int mode, int colour,
                               int S, int tau_q, int32_t *disp_wta, cudaStream_t st)
{
    const long threads = (long)g.B * g.H * g.Wc * g.G;
    const unsigned nb = (unsigned)((threads + 255) / 256);
    const uint32_t SS = (uint32_t)S | ((uint32_t)S << 16);
    const uint32_t TT = (uint32_t)tau_q | ((uint32_t)tau_q << 16);
    const bool pad = (g.L % CH) != 0 || g.G != g.nch;
    const bool wta = disp_wta != nullptr;
#define VSBP_FAST(TD_, MODE_, PAD_, WTA_)                                                                        \
    k_update_fast<TD_, MODE_, PAD_, WTA_><<<nb, 256, 0, st>>>((const TD_ *)D, (uint8_t *)M, (const uint8_t *)Mp, \
                                                               g, colour, SS, TT, disp_wta)
#define VSBP_FAST_PW(TD_, MODE_)                                   \
    if (pad) {                                                     \
        if (wta) VSBP_FAST(TD_, MODE_, true, true);                \
        else VSBP_FAST(TD_, MODE_, true, false);                   \
    } else {                                                       \
        if (wta) VSBP_FAST(TD_, MODE_, false, true);               \
        else VSBP_FAST(TD_, MODE_, false, false);                  \
    }
#define VSBP_FAST_M(TD_)                 \
    if (mode == 0) { VSBP_FAST_PW(TD_, 0) } \
    else if (mode == 1) { VSBP_FAST_PW(TD_, 1) } \
    else { VSBP_FAST_PW(TD_, 2) }
    if (dbytes == 1) {
        VSBP_FAST_M(uint8_t)
    } else {
        VSBP_FAST_M(uint16_t)
    }
#undef VSBP_FAST_M
#undef VSBP_FAST_PW
#undef VSBP_FAST
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
