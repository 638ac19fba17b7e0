// bp_fast.cu -- the packed message-update kernel (row a4, the hot loop), sm_100a.
//
// Same operation as k_update (bp_kernels.cu): one checkerboard colour of min-sum
// messages (Eq.1; R-9..R-12), bit-exact, specialised for the common
// parameter domain (checked on the host, vsbp_api.cu use_fast()):
//   * u8 message storage (tau_q <= 255) and S = 128, so tau_q <= 2S and the
//     truncated-linear lower envelope is an exact 3-tap stencil:
//       m(d) = min(h'(d), h'(d-1) + S, h'(d+1) + S),  h' = min(h - min h, tau_q)
//     (terms |d-d'| >= 2 cost >= 2S >= tau_q; clamping h' at tau_q does not change
//     min(., tau_q), and every stencil term is <= h'(d) <= tau_q);
//   * every belief of the level fits 16 bits (D_max + 4*255 < 2^16), so two labels
//     travel in one 32-bit register as u16x2 on the DPX 16x2 integer datapath
//     (VIMNMX / VIMNMX3 / VIADDMNMX .16x2; plain IADD3 on non-negative halves;
//     PRMT for u8 <-> u16x2).  When beliefs also fit 15 bits (SIGNED) the
//     normalise-and-clamp is one signed VIADDMNMX: min(h + (-min h), tau_q).
// Register j of a thread's 16-label chunk holds (label d0+j, label d0+j+8); the
// storage order of vsbp_internal.cuh makes that a single PRMT per register.
// Labels across chunks come from the adjacent lanes (2 shuffles per pair of
// directions); min_d h reduces over the G lanes (two directions per shuffle).
// Addressing: one 64-bit base per pair, then 32-bit offsets; in the colour-split
// layout the four incoming messages sit at constant offsets from the pixel's own
// row offset.  Slots toward missing neighbours are never read (R-11), so they
// are not zeroed here; the parent read of the first iteration masks them (R-12).
//
// WTA (a5) is fused into the last iteration of level 0 for the colour updated
// there (its belief D + sum of 4 incoming is in registers); MODE 3 computes only
// the WTA (no messages) for the other colour.  HBM traffic per updated pixel:
// L*w_D + 8L bytes (MODE 3: L*w_D + 4L).
#include <type_traits>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel)
{
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

__device__ __forceinline__ uint32_t iadd3(uint32_t a, uint32_t b, uint32_t c) { return a + b + c; }

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

// level-0 data term computed from the grey images instead of read from D_0 (the
// TD = ImgD instantiation): R-2 / R-8, D(x,y,d) = lambda_q * min(|L(x,y) - R(x-d,y)|,
// tau_d) or lambda_q * tau_d for x - d < 0.  The 16 right-image bytes R(x-d0-15 ..
// x-d0) come in as four funnel-aligned words; VABSDIFF4 gives four |L - R| per
// instruction, byte pairs (d0+j, d0+j+8) are gathered into u16x2 with PRMT, then
// min(., tau_d) (VIMNMX.U16x2) and one packed IMAD by lambda_q.  Per updated pixel
// this replaces L bytes of D_0 traffic by ~2 bytes of (L1-resident) image.
struct ImgD {};

__device__ __forceinline__ void dimg_load(const FastArgs &a, int b, int x, int y, int d0, uint32_t dv[8])
{
    const size_t row = ((size_t)b * a.H + y) * (size_t)a.W;
    const int l = __ldg(a.gl + row + x);
    const int a0 = x - d0 - 15;  // first right-image column needed
    if (a0 >= 0 && row + (size_t)a0 + 20 <= a.img_elems) {
        const uintptr_t pa = (uintptr_t)(a.gr + row + a0);
        const uint32_t *wp = reinterpret_cast<const uint32_t *>(pa & ~(uintptr_t)3);
        const uint32_t sh = (uint32_t)(pa & 3) * 8u;
        const uint32_t w0 = __ldg(wp), w1 = __ldg(wp + 1), w2 = __ldg(wp + 2), w3 = __ldg(wp + 3);
        const uint32_t w4 = sh ? __ldg(wp + 4) : 0u;
        const uint32_t l4 = (uint32_t)l * 0x01010101u;
        // D_k byte c = |L - R(a0 + 4k + c)| = label d0 + 15 - 4k - c
        const uint32_t D0 = __vabsdiffu4(l4, __funnelshift_r(w0, w1, sh));
        const uint32_t D1 = __vabsdiffu4(l4, __funnelshift_r(w1, w2, sh));
        const uint32_t D2 = __vabsdiffu4(l4, __funnelshift_r(w2, w3, sh));
        const uint32_t D3 = __vabsdiffu4(l4, __funnelshift_r(w3, w4, sh));
        const uint32_t E0 = D0 & 0x00FF00FFu, O0 = (D0 >> 8) & 0x00FF00FFu;
        const uint32_t E1 = D1 & 0x00FF00FFu, O1 = (D1 >> 8) & 0x00FF00FFu;
        const uint32_t E2 = D2 & 0x00FF00FFu, O2 = (D2 >> 8) & 0x00FF00FFu;
        const uint32_t E3 = D3 & 0x00FF00FFu, O3 = (D3 >> 8) & 0x00FF00FFu;
        const uint32_t pr[8] = {prmt(O3, O1, 0x7632), prmt(E3, E1, 0x7632), prmt(O3, O1, 0x5410),
                                prmt(E3, E1, 0x5410), prmt(O2, O0, 0x7632), prmt(E2, E0, 0x7632),
                                prmt(O2, O0, 0x5410), prmt(E2, E0, 0x5410)};
#pragma unroll
        for (int j = 0; j < 8; ++j) dv[j] = __vminu2(pr[j], a.T2d) * a.lam;
    } else {
        // left image border (x - d < 0 -> lambda_q * tau_d) or the buffer's last bytes
        const uint32_t border = a.lam * (a.T2d & 0xFFFFu);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t c[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int d = d0 + j + 8 * h, xr = x - d;
                c[h] = xr >= 0 ? a.lam * (uint32_t)min(abs(l - (int)__ldg(a.gr + row + xr)), (int)(a.T2d & 0xFFFFu))
                               : border;
            }
            dv[j] = c[0] | (c[1] << 16);
        }
    }
}

// min over the 16 labels of a chunk (both halves), replicated in both halves
__device__ __forceinline__ uint32_t chunk_min(const uint32_t h[8])
{
    const uint32_t a = __vimin3_u16x2(h[0], h[1], h[2]);
    const uint32_t c = __vimin3_u16x2(h[3], h[4], h[5]);
    const uint32_t d = __vimin3_u16x2(a, c, __vminu2(h[6], h[7]));
    return __vminu2(d, prmt(d, 0u, 0x1032));
}

// min over the 16 labels of two chunks: h0's in the low half, h1's in the high half
__device__ __forceinline__ uint32_t chunk_min2(const uint32_t h0[8], const uint32_t h1[8])
{
    const uint32_t a0 = __vimin3_u16x2(__vimin3_u16x2(h0[0], h0[1], h0[2]), __vimin3_u16x2(h0[3], h0[4], h0[5]),
                                       __vminu2(h0[6], h0[7]));
    const uint32_t a1 = __vimin3_u16x2(__vimin3_u16x2(h1[0], h1[1], h1[2]), __vimin3_u16x2(h1[3], h1[4], h1[5]),
                                       __vminu2(h1[6], h1[7]));
    return __vminu2(prmt(a0, a1, 0x5410), prmt(a0, a1, 0x7632));
}

// The 3-tap truncated-linear envelope of a normalised chunk h (every half <= TT):
// out_j = min(h_j, h_{j-1} + S, h_{j+1} + S).  h + S is formed with a plain 32-bit add
// (no carry between the halves: TT + S < 2^16), which the compiler may put on the FMA
// pipe, then one 3-input u16x2 min per word on the ALU pipe -- instead of two
// add-min (VIADDMNMX) ALU instructions per word.  The lane-boundary neighbours `pv0`
// (label d0-1, in the half matching e) and `nx7` (d0+16) arrive already offset by S.
__device__ __forceinline__ void envelope(const uint32_t h[8], const uint32_t hs[8], uint32_t prev0s,
                                         uint32_t next7s, uint32_t out[8])
{
#pragma unroll
    for (int j = 0; j < 8; ++j)
        out[j] = __vimin3_u16x2(h[j], j == 0 ? prev0s : hs[j - 1], j == 7 ? next7s : hs[j + 1]);
}

// WTA (a5) from the five belief terms of a chunk when every belief is below 2^12
// (u8 costs: D + 4 tau_q <= 255 + 4 * 255): each u16 half becomes cost * 16 + its label
// offset in the chunk (j, or j + 8 in the high half), formed by one multiply-add, so a
// u16x2 min tree finds the minimum cost with the smallest label among equal costs;
// the lanes then reduce (cost << 9 | label) keys.  Same result as wta_key.
template <bool PAD>
__device__ __forceinline__ uint32_t wta_key16(const uint32_t dv[8], const uint32_t (&in)[4][8], int d0, int L, int G)
{
    uint32_t k[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t tot = iadd3(dv[j], in[0][j], in[1][j]) + in[2][j] + in[3][j];
        k[j] = tot * 16u + ((uint32_t)j | ((uint32_t)(j + 8) << 16));  // no carry between halves
        if (PAD) k[j] |= (d0 + j >= L ? 0x0000FFFFu : 0u) | (d0 + j + 8 >= L ? 0xFFFF0000u : 0u);
    }
    const uint32_t m = __vimin3_u16x2(__vimin3_u16x2(k[0], k[1], k[2]), __vimin3_u16x2(k[3], k[4], k[5]),
                                      __vminu2(k[6], k[7]));
    const uint32_t k16 = min(m & 0xFFFFu, m >> 16);  // low-half labels are the smaller ones
    uint32_t best = ((k16 >> 4) << 9) | (uint32_t)d0 | (k16 & 15u);
    for (int s = G >> 1; s > 0; s >>= 1) best = min(best, __shfl_xor_sync(FULL, best, s, G));
    return best & 511u;
}

// MODE 0: normal iteration; 1: top level t=0 (all incoming 0); 2: lower level t=0
// (incoming read from the parent level); 3: WTA only (no message update).
// PAD: some labels of the chunk are >= L.  WTA: write the WTA label of the pixel.
// SIGNED: beliefs < 2^15, normalise+clamp in one signed VIADDMNMX.
template <typename TD, int MODE, bool PAD, bool WTA, bool SIGNED>
__global__ void __launch_bounds__(256, 4) k_update_fast(FastArgs a, const TD *__restrict__ D)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    const int lane_g = threadIdx.x & (a.G - 1);
    const uint32_t pix = t >> a.log2G;
    bool active = pix < a.npix;
    if (__all_sync(FULL, !active)) return;
    const uint32_t y = a.magic ? __umulhi(pix, a.magic) : pix / (uint32_t)a.Wc;
    const uint32_t i = pix - y * (uint32_t)a.Wc;
    const uint32_t o = (a.colour + y) & 1u;
    const int x = 2 * (int)i + (int)o;
    active = active && x < a.W;
    const bool io = active && lane_g < a.nch;
    const int d0 = lane_g * CH;
    const bool has[4] = {y > 0, (int)y < a.H - 1, x > 0, x < a.W - 1};

    const uint32_t P = a.plane;                          // H * Wc * Lp
    const uint32_t r = (y * (uint32_t)a.Wc + i) * (uint32_t)a.Lp + (uint32_t)d0;
    const uint32_t rowstep = (uint32_t)a.Wc * (uint32_t)a.Lp;
    uint8_t *Mb = a.M + (size_t)b * a.pairM;

    // ---- loads: incoming messages (neighbour in direction k sends on slot k^1)
    uint4 wi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) wi[k] = make_uint4(0u, 0u, 0u, 0u);
    if (MODE == 0 || MODE == 3) {
        const uint8_t *Mo = Mb + (size_t)((a.colour ^ 1) * 4u) * P;
        if (io && has[0]) wi[0] = __ldg(reinterpret_cast<const uint4 *>(Mo + (1u * P + r - rowstep)));
        if (io && has[1]) wi[1] = __ldg(reinterpret_cast<const uint4 *>(Mo + (r + rowstep)));
        if (io && has[2]) wi[2] = __ldg(reinterpret_cast<const uint4 *>(Mo + (3u * P + r + (o - 1u) * (uint32_t)a.Lp)));
        if (io && has[3]) wi[3] = __ldg(reinterpret_cast<const uint4 *>(Mo + (2u * P + r + o * (uint32_t)a.Lp)));
    } else if (MODE == 2) {
        const uint8_t *Mpb = a.Mp + (size_t)b * a.pairMp;
        // neighbour k's parent (px, py) sends on slot k^1; vertical neighbours share
        // the pixel's parent column, horizontal ones its parent row
        const int X = x >> 1, Y = (int)y >> 1;
        const int pyu = ((int)y - 1) >> 1, pyd = ((int)y + 1) >> 1, pxl = (x - 1) >> 1, pxr = (x + 1) >> 1;
        const uint32_t Lp = (uint32_t)a.Lp, Wcp = (uint32_t)a.Wcp;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int px = k == 2 ? pxl : (k == 3 ? pxr : X);
            const int py = k == 0 ? pyu : (k == 1 ? pyd : Y);
            const int slot = k ^ 1;
            // R-12: the parent's slot toward a missing neighbour counts as 0
            const bool ph = slot == 0 ? py > 0 : slot == 1 ? py < a.Hp - 1 : slot == 2 ? px > 0 : px < a.Wp - 1;
            const uint32_t off = ((uint32_t)(((px + py) & 1) * 4 + slot)) * a.planep +
                                 ((uint32_t)py * Wcp + (uint32_t)(px >> 1)) * Lp + (uint32_t)d0;
            if (io && has[k] && ph) wi[k] = __ldg(reinterpret_cast<const uint4 *>(Mpb + off));
        }
    }
    uint32_t dv[8];
    if (io) {
        if constexpr (std::is_same<TD, ImgD>::value)
            dimg_load(a, b, x, (int)y, d0, dv);
        else
            DLoad<TD>::load(D + (size_t)b * a.pairD + a.colour * P + r, dv);
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) dv[j] = 0u;
    }
    uint32_t in[4][8];
#pragma unroll
    for (int k = 0; k < 4; ++k) unpack_u8(wi[k], in[k]);

    // ---- fused WTA (a5): argmin of the belief D + sum of the 4 incoming, ties -> smallest d
    if (WTA && sizeof(TD) == 1) {  // u8 costs (or the image data term, <= 255): beliefs < 2^12
        const uint32_t lab = wta_key16<PAD>(dv, in, d0, a.L, a.G);
        if (active && lane_g == 0) a.disp[((size_t)b * a.H + y) * a.W + x] = (int32_t)lab;
    } else if (WTA) {
        uint32_t best = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t tot = iadd3(dv[j], in[0][j], in[1][j]) + in[2][j] + in[3][j];
            const uint32_t lo = tot & 0xFFFFu, hi = tot >> 16;
            if (!PAD || d0 + j < a.L) best = min(best, (lo << 9) | (uint32_t)(d0 + j));
            if (!PAD || d0 + j + 8 < a.L) best = min(best, (hi << 9) | (uint32_t)(d0 + j + 8));
        }
        for (int s = a.G >> 1; s > 0; s >>= 1) best = min(best, __shfl_xor_sync(FULL, best, s, a.G));
        if (active && lane_g == 0) a.disp[((size_t)b * a.H + y) * a.W + x] = (int32_t)(best & 511u);
    }
    if (MODE == 3) return;

    uint32_t padm[8];
    if (PAD) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            padm[j] = (d0 + j >= a.L ? (SIGNED ? 0x00007FFFu : 0x0000FFFFu) : 0u) |
                      (d0 + j + 8 >= a.L ? (SIGNED ? 0x7FFF0000u : 0xFFFF0000u) : 0u);
    }

    // ---- the four outgoing messages, two directions at a time:
    //      h_0 = D + in1+in2+in3, h_1 = D + in0+in2+in3 share D+in2+in3, etc.
#pragma unroll
    for (int kp = 0; kp < 4; kp += 2) {
        uint32_t h[2][8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t base = kp == 0 ? iadd3(dv[j], in[2][j], in[3][j]) : iadd3(dv[j], in[0][j], in[1][j]);
            h[0][j] = base + in[kp + 1][j];
            h[1][j] = base + in[kp][j];
            if (PAD) {
                h[0][j] |= padm[j];
                h[1][j] |= padm[j];
            }
        }
        // min over the G lanes: direction kp in the low half, kp+1 in the high half
        uint32_t pm = chunk_min2(h[0], h[1]);
        for (int s = a.G >> 1; s > 0; s >>= 1) pm = __vminu2(pm, __shfl_xor_sync(FULL, pm, s, a.G));
        // h' = min(h - min h, tau_q), and h' + S for the envelope
        uint32_t hs[2][8];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const uint32_t hm = prmt(pm, 0u, e == 0 ? 0x1010 : 0x3232);
            if (SIGNED) {
                const uint32_t neg = prmt(0u - hm, 0u, 0x1010);  // (-min h) as s16 in both halves
#pragma unroll
                for (int j = 0; j < 8; ++j) h[e][j] = (uint32_t)__viaddmin_s16x2(h[e][j], neg, a.TT);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) h[e][j] = __vminu2(h[e][j] - hm, a.TT);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) hs[e][j] = h[e][j] + a.SS;
        }
        // labels d0-1 (lane-1's r7 high half) and d0+16 (lane+1's r0 low half), + S
        uint32_t up = __shfl_up_sync(FULL, prmt(hs[0][7], hs[1][7], 0x7632), 1, a.G);
        uint32_t dn = __shfl_down_sync(FULL, prmt(hs[0][0], hs[1][0], 0x5410), 1, a.G);
        if (lane_g == 0) up = a.TT;
        if (lane_g == a.G - 1) dn = a.TT;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            uint32_t out[8];
            envelope(h[e], hs[e], prmt(up, hs[e][7], e == 0 ? 0x5410 : 0x5432),  // (d0-1, d0+7)
                     prmt(hs[e][0], dn, e == 0 ? 0x5432 : 0x7632), out);          // (d0+8, d0+16)
            if (PAD) {
#pragma unroll
                for (int j = 0; j < 8; ++j) out[j] &= ~padm[j];
            }
            if (io)
                *reinterpret_cast<uint4 *>(Mb + ((a.colour * 4u + (uint32_t)(kp + e)) * P + r)) = pack_u8(out);
        }
    }
}

// ---------------------------------------------------------------- fused final iteration (a4 + a5)
// The last level-0 iteration updates colour A and is followed only by the WTA of
// both colours, so its messages are consumed once, by the WTA of their receivers.
// k_final_fast therefore never stores them: one G-lane group per colour-B pixel p
// computes the four messages m_{q->p} of its colour-A neighbours q itself (the same
// arithmetic as k_update_fast: h_q = D_q + the three incoming of q other than p's,
// normalise, 3-tap envelope), adds them to D_p and takes p's WTA; the group also
// labels its right neighbour q (belief h_q + m_{p->q}), and the pixel at x = 1 its
// left neighbour (x = 0), so every colour-A pixel is labelled exactly once.
// HBM per pixel pair: D_A, D_B and the four colour-B message planes (6L bytes at
// u8) instead of 9L (last update) + 5L (WTA of the other colour); each colour-A
// pixel's data is re-read by its four neighbours from L1/L2.  Requires W >= 2.
template <bool PAD, bool SIGNED>
__device__ __forceinline__ void one_message(const FastArgs &a, uint32_t h[8], const uint32_t padm[8], int lane_g,
                                            uint32_t out[8])
{
    uint32_t m = chunk_min(h);
    for (int s = a.G >> 1; s > 0; s >>= 1) m = __vminu2(m, __shfl_xor_sync(FULL, m, s, a.G));
    if (SIGNED) {
        const uint32_t neg = prmt(0u - m, 0u, 0x1010);
#pragma unroll
        for (int j = 0; j < 8; ++j) h[j] = (uint32_t)__viaddmin_s16x2(h[j], neg, a.TT);
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) h[j] = __vminu2(h[j] - m, a.TT);
    }
    uint32_t up = __shfl_up_sync(FULL, h[7], 1, a.G);
    uint32_t dn = __shfl_down_sync(FULL, h[0], 1, a.G);
    if (lane_g == 0) up = a.TT;
    if (lane_g == a.G - 1) dn = a.TT;
    const uint32_t prev0 = prmt(up, h[7], 0x5432);  // (d0-1, d0+7)
    const uint32_t next7 = prmt(h[0], dn, 0x5432);  // (d0+8, d0+16)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t pv = j == 0 ? prev0 : h[j - 1];
        const uint32_t nx = j == 7 ? next7 : h[j + 1];
        out[j] = __viaddmin_u16x2(pv, a.SS, __viaddmin_u16x2(nx, a.SS, h[j]));
        if (PAD) out[j] &= ~padm[j];
    }
}

template <bool PAD>
__device__ __forceinline__ uint32_t wta_key(const uint32_t tot[8], int d0, int L, int G)
{
    uint32_t best = 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t lo = tot[j] & 0xFFFFu, hi = tot[j] >> 16;
        if (!PAD || d0 + j < L) best = min(best, (lo << 9) | (uint32_t)(d0 + j));
        if (!PAD || d0 + j + 8 < L) best = min(best, (hi << 9) | (uint32_t)(d0 + j + 8));
    }
    for (int s = G >> 1; s > 0; s >>= 1) best = min(best, __shfl_xor_sync(FULL, best, s, G));
    return best & 511u;
}

template <bool PAD, bool SIGNED>
__global__ void __launch_bounds__(256, 4) k_final_fast(FastArgs a, const uint8_t *__restrict__ D)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    const int lane_g = threadIdx.x & (a.G - 1);
    const uint32_t pix = t >> a.log2G;
    bool active = pix < a.npix;
    if (__all_sync(FULL, !active)) return;
    const uint32_t cA = a.colour, cB = a.colour ^ 1u;
    const uint32_t y = a.magic ? __umulhi(pix, a.magic) : pix / (uint32_t)a.Wc;
    const uint32_t i = pix - y * (uint32_t)a.Wc;
    const uint32_t o = (cB + y) & 1u;
    const int x = 2 * (int)i + (int)o;
    active = active && x < a.W;
    const bool io = active && lane_g < a.nch;
    const int d0 = lane_g * CH;
    const uint32_t P = a.plane;
    const uint32_t rowstep = (uint32_t)a.Wc * (uint32_t)a.Lp;
    const uint32_t r = (y * (uint32_t)a.Wc + i) * (uint32_t)a.Lp + (uint32_t)d0;
    const uint8_t *Mb = a.M + (size_t)b * a.pairM;
    const uint8_t *MB = Mb + (size_t)(cB * 4u) * P;  // colour-B senders: the incoming of every A pixel
    const uint8_t *Db = D + (size_t)b * a.pairD;

    uint32_t padm[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        padm[j] = !PAD ? 0u
                       : (d0 + j >= a.L ? (SIGNED ? 0x00007FFFu : 0x0000FFFFu) : 0u) |
                             (d0 + j + 8 >= a.L ? (SIGNED ? 0x7FFF0000u : 0xFFFF0000u) : 0u);
    uint32_t bel[8];
    {
        uint4 w = make_uint4(0u, 0u, 0u, 0u);
        if (io) w = __ldg(reinterpret_cast<const uint4 *>(Db + cB * P + r));
        unpack_u8(w, bel);
    }
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
        const bool has = k == 0 ? y > 0 : k == 1 ? (int)y < a.H - 1 : k == 2 ? x > 0 : x < a.W - 1;
        if (__all_sync(FULL, !has)) continue;
        // neighbour q (colour A) and the direction kk from q to p
        const int xq = x + (k == 2 ? -1 : (k == 3 ? 1 : 0));
        const int yq = (int)y + (k == 0 ? -1 : (k == 1 ? 1 : 0));
        const uint32_t oq = (cA + (uint32_t)yq) & 1u;
        const uint32_t iq = (uint32_t)(xq - (int)oq) >> 1;
        const uint32_t rq = ((uint32_t)yq * (uint32_t)a.Wc + iq) * (uint32_t)a.Lp + (uint32_t)d0;
        const int kk = k ^ 1;
        const bool hq[4] = {yq > 0, yq < a.H - 1, xq > 0, xq < a.W - 1};
        const bool ld = io && has;
        uint4 wi[4], wd = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) wi[k2] = make_uint4(0u, 0u, 0u, 0u);
        // the incoming of q (its neighbour in direction k2 sends on slot k2^1); q's
        // incoming from p itself (k2 == kk) is loaded only for q's WTA below
        const bool wq = k == 3 || (k == 2 && xq == 0);  // this group labels q
        if (ld && hq[0] && (kk != 0 || wq)) wi[0] = __ldg(reinterpret_cast<const uint4 *>(MB + (1u * P + rq - rowstep)));
        if (ld && hq[1] && (kk != 1 || wq)) wi[1] = __ldg(reinterpret_cast<const uint4 *>(MB + (rq + rowstep)));
        if (ld && hq[2] && (kk != 2 || wq)) wi[2] = __ldg(reinterpret_cast<const uint4 *>(MB + (3u * P + rq + (oq - 1u) * (uint32_t)a.Lp)));
        if (ld && hq[3] && (kk != 3 || wq)) wi[3] = __ldg(reinterpret_cast<const uint4 *>(MB + (2u * P + rq + oq * (uint32_t)a.Lp)));
        if (ld) wd = __ldg(reinterpret_cast<const uint4 *>(Db + cA * P + rq));
        uint32_t dq[8], in[4][8];
        unpack_u8(wd, dq);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) unpack_u8(wi[k2], in[k2]);
        // h_q without p's message: sum the three other directions
        uint32_t h[8], pin[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t all4 = iadd3(dq[j], in[0][j], in[1][j]) + in[2][j] + in[3][j];
            pin[j] = kk == 0 ? in[0][j] : kk == 1 ? in[1][j] : kk == 2 ? in[2][j] : in[3][j];
            h[j] = all4 - pin[j];
        }
        if (__any_sync(FULL, wq && has)) {
            // label q: belief D_q + all four incoming = h + p's message
            uint32_t tot[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) tot[j] = h[j] + pin[j];
            const uint32_t lab = wta_key<PAD>(tot, d0, a.L, a.G);
            if (wq && has && active && lane_g == 0) a.disp[((size_t)b * a.H + yq) * a.W + xq] = (int32_t)lab;
        }
        if (PAD) {
#pragma unroll
            for (int j = 0; j < 8; ++j) h[j] |= padm[j];
        }
        uint32_t m[8];
        one_message<PAD, SIGNED>(a, h, padm, lane_g, m);
        if (has) {
#pragma unroll
            for (int j = 0; j < 8; ++j) bel[j] += m[j];
        }
    }
    const uint32_t lab = wta_key<PAD>(bel, d0, a.L, a.G);
    if (active && lane_g == 0) a.disp[((size_t)b * a.H + y) * a.W + x] = (int32_t)lab;
}

// ---------------------------------------------------------------- fused final iteration, tiled
// k_final_tile: the same fusion as k_final_fast without the recomputation.  A CTA
// owns a tile of TY rows x TX colour-columns of colour-B pixels and the colour-A
// pixels with the same coordinates.  Phase 1 updates every colour-A pixel adjacent
// to the tile (the owned ones, the unowned column on the side the row's parity
// needs, and the rows above and below -- vertical messages only) exactly like
// k_update_fast, but keeps the packed u8 messages in shared memory; owned pixels
// are labelled from D + the four incoming.  Phase 2 labels each colour-B pixel of
// the tile from D_B + its four messages read from shared memory.  HBM per pixel
// pair ~ (1 + halo) * 5L + L instead of 14L; nothing but labels is written.
constexpr int FT_TY = 8, FT_TX = 16;

template <bool PAD, bool SIGNED>
__global__ void __launch_bounds__(256, 3) k_final_tile(FastArgs a, const uint8_t *__restrict__ D)
{
    extern __shared__ uint4 fsm[];  // [(TY+2)*(TX+2)][4][nch] packed u8 chunks
    const int b = blockIdx.z;
    const int G = a.G, nch = a.nch;
    const int lane_g = threadIdx.x & (G - 1);
    const int grp = threadIdx.x >> a.log2G, ngrp = blockDim.x >> a.log2G;
    const int y0 = blockIdx.y * FT_TY, i0 = blockIdx.x * FT_TX;
    const uint32_t cA = a.colour, cB = a.colour ^ 1u;
    const bool io_lane = lane_g < nch;
    const int d0 = lane_g * CH;
    const uint32_t P = a.plane;
    const uint32_t rowstep = (uint32_t)a.Wc * (uint32_t)a.Lp;
    const uint8_t *Mb = a.M + (size_t)b * a.pairM;
    const uint8_t *MB = Mb + (size_t)(cB * 4u) * P;
    const uint8_t *Db = D + (size_t)b * a.pairD;
    constexpr int NA = (FT_TY + 2) * (FT_TX + 2);
    uint32_t padm[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        padm[j] = !PAD ? 0u
                       : (d0 + j >= a.L ? (SIGNED ? 0x00007FFFu : 0x0000FFFFu) : 0u) |
                             (d0 + j + 8 >= a.L ? (SIGNED ? 0x7FFF0000u : 0xFFFF0000u) : 0u);

    // ---- phase 1: colour-A pixels around the tile (warp-uniform trip count)
    for (int base = 0; base < NA; base += ngrp) {
        const int task = base + grp;
        const int tya = task / (FT_TX + 2), txa = task - tya * (FT_TX + 2);
        const int ya = y0 - 1 + tya, ia = i0 - 1 + txa;
        const uint32_t oa = (cA + (uint32_t)ya) & 1u;
        const int xa = 2 * ia + (int)oa;
        const bool inimg = task < NA && ya >= 0 && ya < a.H && ia >= 0 && ia < a.Wc && xa < a.W;
        const bool rowin = tya >= 1 && tya <= FT_TY;
        // the B pixels of row ya have parity oB = 1 - oa: their A neighbours span
        // colour-columns [i0 + oB - 1, i0 + TX + oB - 1]
        const int lo_t = oa ? 0 : 1;  // first needed txa in a tile row
        const bool need_h = rowin && txa >= lo_t && txa <= lo_t + FT_TX;
        const bool need_v = txa >= 1 && txa <= FT_TX;  // rows y0-1 .. y0+TY
        const bool owned = rowin && txa >= 1 && txa <= FT_TX;
        const bool act = inimg && (need_h || need_v);
        const bool io = act && io_lane;
        const uint32_t r = ((uint32_t)ya * (uint32_t)a.Wc + (uint32_t)ia) * (uint32_t)a.Lp + (uint32_t)d0;
        const bool has[4] = {ya > 0, ya < a.H - 1, xa > 0, xa < a.W - 1};
        uint4 wi[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) wi[k] = make_uint4(0u, 0u, 0u, 0u);
        if (io && has[0]) wi[0] = __ldg(reinterpret_cast<const uint4 *>(MB + (1u * P + r - rowstep)));
        if (io && has[1]) wi[1] = __ldg(reinterpret_cast<const uint4 *>(MB + (r + rowstep)));
        if (io && has[2]) wi[2] = __ldg(reinterpret_cast<const uint4 *>(MB + (3u * P + r + (oa - 1u) * (uint32_t)a.Lp)));
        if (io && has[3]) wi[3] = __ldg(reinterpret_cast<const uint4 *>(MB + (2u * P + r + oa * (uint32_t)a.Lp)));
        uint4 wd = make_uint4(0u, 0u, 0u, 0u);
        if (io) wd = __ldg(reinterpret_cast<const uint4 *>(Db + cA * P + r));
        uint32_t dv[8], in[4][8];
        unpack_u8(wd, dv);
#pragma unroll
        for (int k = 0; k < 4; ++k) unpack_u8(wi[k], in[k]);
        if (__any_sync(FULL, owned && act)) {
            uint32_t tot[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) tot[j] = iadd3(dv[j], in[0][j], in[1][j]) + in[2][j] + in[3][j];
            const uint32_t lab = wta_key<PAD>(tot, d0, a.L, G);
            if (owned && inimg && lane_g == 0) a.disp[((size_t)b * a.H + ya) * a.W + xa] = (int32_t)lab;
        }
        uint4 *slot = fsm + (size_t)task * 4 * nch + lane_g;
#pragma unroll
        for (int kp = 0; kp < 4; kp += 2) {
            if (!__any_sync(FULL, act && (kp == 0 ? need_v : need_h))) continue;
            uint32_t h[2][8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t bs = kp == 0 ? iadd3(dv[j], in[2][j], in[3][j]) : iadd3(dv[j], in[0][j], in[1][j]);
                h[0][j] = bs + in[kp + 1][j];
                h[1][j] = bs + in[kp][j];
                if (PAD) {
                    h[0][j] |= padm[j];
                    h[1][j] |= padm[j];
                }
            }
            uint32_t pm = prmt(chunk_min(h[0]), chunk_min(h[1]), 0x5410);
            for (int s2 = G >> 1; s2 > 0; s2 >>= 1) pm = __vminu2(pm, __shfl_xor_sync(FULL, pm, s2, G));
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t hm = prmt(pm, 0u, e == 0 ? 0x1010 : 0x3232);
                if (SIGNED) {
                    const uint32_t neg = prmt(0u - hm, 0u, 0x1010);
#pragma unroll
                    for (int j = 0; j < 8; ++j) h[e][j] = (uint32_t)__viaddmin_s16x2(h[e][j], neg, a.TT);
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) h[e][j] = __vminu2(h[e][j] - hm, a.TT);
                }
            }
            uint32_t up = __shfl_up_sync(FULL, prmt(h[0][7], h[1][7], 0x7632), 1, G);
            uint32_t dn = __shfl_down_sync(FULL, prmt(h[0][0], h[1][0], 0x5410), 1, G);
            if (lane_g == 0) up = a.TT;
            if (lane_g == G - 1) dn = a.TT;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t prev0 = prmt(up, h[e][7], e == 0 ? 0x5410 : 0x5432);
                const uint32_t next7 = prmt(h[e][0], dn, e == 0 ? 0x5432 : 0x7632);
                uint32_t out[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t pv = j == 0 ? prev0 : h[e][j - 1];
                    const uint32_t nx = j == 7 ? next7 : h[e][j + 1];
                    out[j] = __viaddmin_u16x2(pv, a.SS, __viaddmin_u16x2(nx, a.SS, h[e][j]));
                    if (PAD) out[j] &= ~padm[j];
                }
                if (io && (kp == 0 ? need_v : need_h)) slot[(kp + e) * nch] = pack_u8(out);
            }
        }
    }
    __syncthreads();

    // ---- phase 2: colour-B pixels of the tile
    for (int base = 0; base < FT_TY * FT_TX; base += ngrp) {
        const int bt = base + grp;
        const int ty = bt / FT_TX, tx = bt - ty * FT_TX;
        const int y = y0 + ty, ib = i0 + tx;
        const uint32_t ob = (cB + (uint32_t)y) & 1u;
        const int x = 2 * ib + (int)ob;
        const bool act = bt < FT_TY * FT_TX && y < a.H && ib < a.Wc && x < a.W;
        const bool io = act && io_lane;
        const uint32_t r = ((uint32_t)y * (uint32_t)a.Wc + (uint32_t)ib) * (uint32_t)a.Lp + (uint32_t)d0;
        uint4 wd = make_uint4(0u, 0u, 0u, 0u);
        if (io) wd = __ldg(reinterpret_cast<const uint4 *>(Db + cB * P + r));
        uint32_t bel[8];
        unpack_u8(wd, bel);
        const bool has[4] = {y > 0, y < a.H - 1, x > 0, x < a.W - 1};
        // neighbour k's tile slot and the direction it sends toward this pixel
        const int sl[4] = {ty * (FT_TX + 2) + tx + 1, (ty + 2) * (FT_TX + 2) + tx + 1,
                           (ty + 1) * (FT_TX + 2) + tx + (int)ob, (ty + 1) * (FT_TX + 2) + tx + (int)ob + 1};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!(io && has[k])) continue;
            uint32_t m[8];
            unpack_u8(fsm[((size_t)sl[k] * 4 + (k ^ 1)) * nch + lane_g], m);
#pragma unroll
            for (int j = 0; j < 8; ++j) bel[j] += m[j];
        }
        const uint32_t lab = wta_key<PAD>(bel, d0, a.L, G);
        if (act && lane_g == 0) a.disp[((size_t)b * a.H + y) * a.W + x] = (int32_t)lab;
    }
}

size_t final_tile_smem(int nch) { return (size_t)(FT_TY + 2) * (FT_TX + 2) * 4 * nch * sizeof(uint4); }

cudaError_t launch_final_tile(const void *D, const FastArgs &a, int B, bool sgn, cudaStream_t st)
{
    const size_t smem = final_tile_smem(a.nch);
    const bool pad = (a.L % CH) != 0 || a.G != a.nch;
    static bool attr = false;
    if (!attr) {
        const void *fs[] = {(const void *)k_final_tile<false, false>, (const void *)k_final_tile<false, true>,
                            (const void *)k_final_tile<true, false>, (const void *)k_final_tile<true, true>};
        for (const void *f : fs) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            if (e != cudaSuccess) return e;
        }
        attr = true;
    }
    dim3 grid((unsigned)((a.Wc + FT_TX - 1) / FT_TX), (unsigned)((a.H + FT_TY - 1) / FT_TY), (unsigned)B);
    const uint8_t *d = (const uint8_t *)D;
    if (pad) {
        if (sgn) k_final_tile<true, true><<<grid, 256, smem, st>>>(a, d);
        else k_final_tile<true, false><<<grid, 256, smem, st>>>(a, d);
    } else {
        if (sgn) k_final_tile<false, true><<<grid, 256, smem, st>>>(a, d);
        else k_final_tile<false, false><<<grid, 256, smem, st>>>(a, d);
    }
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_final_fast(const void *D, const FastArgs &a, int B, bool sgn, cudaStream_t st)
{
    const long threads = (long)a.npix * a.G;
    dim3 grid((unsigned)((threads + 255) / 256), (unsigned)B);
    const bool pad = (a.L % CH) != 0 || a.G != a.nch;
    const uint8_t *d = (const uint8_t *)D;
    if (pad) {
        if (sgn) k_final_fast<true, true><<<grid, 256, 0, st>>>(a, d);
        else k_final_fast<true, false><<<grid, 256, 0, st>>>(a, d);
    } else {
        if (sgn) k_final_fast<false, true><<<grid, 256, 0, st>>>(a, d);
        else k_final_fast<false, false><<<grid, 256, 0, st>>>(a, d);
    }
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- two iterations per launch
// k_update_pair: checkerboard iterations t (colour A = a.colour) and t+1 (colour B)
// in one launch (north_star "several checkerboard iterations per launch";
// DESIGN §8).  The messages colour A sends at iteration t are read by exactly one
// consumer -- colour B's update at t+1 -- and are rewritten at t+2 before anything
// else reads them, so they never go to HBM: a CTA walks down the rows of a band of
// its column tile, and for every row ya
//   A-phase: updates the colour-A pixels of row ya (plus one halo pixel on each
//            side of the tile) from colour B's iteration-(t-1) messages (or from the
//            parent level, MODE 2; or from nothing, MODE 1) and keeps their four
//            outgoing messages in a 3-row shared-memory ring;
//   B-phase: updates the colour-B pixels of row ya-1 from the ring (rows ya-2,
//            ya-1, ya) and writes their messages to the level's OTHER message array
//            (a.Mw): colour-B messages of iteration t-1 are still being read by the
//            neighbouring tiles and bands, so the level's messages ping-pong between
//            two arrays at every fused pair (the host switches its base pointer).
// Per pixel pair HBM carries D_A + D_B + colour-B messages in (4L) and out (4L) --
// 10L bytes at u8 -- instead of 2 x 9L for two single-iteration launches.  The
// arithmetic per pixel is k_update_fast's, so the messages are bit-identical.
// The colour-A halo (2 pixels per 64-pixel tile row, 2 rows per band) is computed
// twice.  Requires TD = u8 / u16 D, u8 messages (the fast-kernel domain).
template <bool PAD, bool SIGNED, int GT, typename Store>
__device__ __forceinline__ void outgoing(const FastArgs &a, const uint32_t dv[8], const uint32_t (&in)[4][8],
                                         const uint32_t padm[8], int lane_g, Store store)
{
    const int G = GT ? GT : a.G;  // lanes per pixel (compile-time for the common L)
#pragma unroll
    for (int kp = 0; kp < 4; kp += 2) {
        uint32_t h[2][8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t base = kp == 0 ? iadd3(dv[j], in[2][j], in[3][j]) : iadd3(dv[j], in[0][j], in[1][j]);
            h[0][j] = base + in[kp + 1][j];
            h[1][j] = base + in[kp][j];
            if (PAD) {
                h[0][j] |= padm[j];
                h[1][j] |= padm[j];
            }
        }
        uint32_t pm = chunk_min2(h[0], h[1]);
#pragma unroll
        for (int s = G >> 1; s > 0; s >>= 1) pm = __vminu2(pm, __shfl_xor_sync(FULL, pm, s, G));
        uint32_t hs[2][8];  // h' + S
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const uint32_t hm = prmt(pm, 0u, e == 0 ? 0x1010 : 0x3232);
            if (SIGNED) {
                const uint32_t neg = prmt(0u - hm, 0u, 0x1010);
#pragma unroll
                for (int j = 0; j < 8; ++j) h[e][j] = (uint32_t)__viaddmin_s16x2(h[e][j], neg, a.TT);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) h[e][j] = __vminu2(h[e][j] - hm, a.TT);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) hs[e][j] = h[e][j] + a.SS;
        }
        // labels d0-1 (lane-1's r7 high half) and d0+16 (lane+1's r0 low half), + S;
        // outside the chunk range TT (>= every h', so no effect)
        uint32_t up = __shfl_up_sync(FULL, prmt(hs[0][7], hs[1][7], 0x7632), 1, G);
        uint32_t dn = __shfl_down_sync(FULL, prmt(hs[0][0], hs[1][0], 0x5410), 1, G);
        if (lane_g == 0) up = a.TT;
        if (lane_g == G - 1) dn = a.TT;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            uint32_t out[8];
            envelope(h[e], hs[e], prmt(up, hs[e][7], e == 0 ? 0x5410 : 0x5432),
                     prmt(hs[e][0], dn, e == 0 ? 0x5432 : 0x7632), out);
            if (PAD) {
#pragma unroll
                for (int j = 0; j < 8; ++j) out[j] &= ~padm[j];
            }
            store(kp + e, out);
        }
    }
}

template <typename TD>
__device__ __forceinline__ void load_d(const TD *p, bool io, uint32_t dv[8])
{
    if (io) {
        DLoad<TD>::load(p, dv);
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) dv[j] = 0u;
    }
}

// CTA size and staging depth of k_update_pair: 128 threads with one
// staging buffer take 44 KB of shared memory (u8 costs), so 5 CTAs (20 warps) fit an
// SM; 256 threads with double buffering (112 KB, 16 warps) measured 10 % slower
#ifndef VSBP_PAIR_T
#define VSBP_PAIR_T 128
#endif
#ifndef VSBP_PAIR_NBUF
#define VSBP_PAIR_NBUF 1
#endif
constexpr int PAIR_T = VSBP_PAIR_T;  // threads per CTA of k_update_pair
// staging buffers: 2 = cp.async into the other buffer while this step reads its own;
// 1 = the step first moves its staged inputs to registers, then refills the buffer
constexpr int PAIR_NBUF = VSBP_PAIR_NBUF;
constexpr int PAIR_MINB = PAIR_T == 256 ? 2 : (PAIR_NBUF == 1 ? 5 : 4);

__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc, bool valid)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gsrc), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Every global input of a row step is prefetched one step ahead with cp.async into
// a per-thread staging slot (no registers held, zero-filled where a neighbour does
// not exist), so the barrier-separated phases never wait on HBM latency:
//   stage[buf][0..3][tid]   the 4 incoming chunks of the thread's colour-A pixel
//   stage[buf][4..4+DW)     its D chunk(s);  stage[buf][4+DW..4+2DW)  the colour-B pixel's
// FIN: the level's LAST iteration (colour A, MODE 0) fused with the WTA (a5) of both
// colours: the A-phase labels its pixels from the staged incoming (the belief is in
// registers), keeps its outgoing messages in the ring, and the B-phase only labels the
// colour-B pixels from them -- no message is written (bp_get_messages(level 0) is then
// unavailable, as with VSBP_OPT_FINAL 1/2).  HBM per pixel pair: D_A + D_B + 4L.
template <typename TD, int MODEA, bool PAD, bool SIGNED, int GT, bool FIN>
__global__ void __launch_bounds__(PAIR_T, PAIR_MINB) k_update_pair(FastArgs a, const TD *__restrict__ D, int band)
{
    const int G = GT ? GT : a.G, LOG2G = GT == 1 ? 0 : GT == 2 ? 1 : GT == 4 ? 2 : GT == 8 ? 3 : a.log2G;
    constexpr int DW = sizeof(TD) == 1 ? 1 : 2;  // 16-byte D chunks per lane
    constexpr int NST = 4 + 2 * DW;
    extern __shared__ uint4 smem[];
    // colour-A messages kept UNPACKED (u16x2, two uint4 per lane: no PRMT pack in the
    // A-phase, no unpack in the B-phase), one buffer per (slot, row) still to be read:
    // slot 0 of row ya (read by B(ya-1) in the same step), slots 2/3 of rows ya and
    // ya-1 (B(ya-1), B(ya)), slot 1 of rows ya-2..ya (B(ya-1), B(ya), B(ya+1))
    // (u16 costs need 2x the staging, so their ring stays packed u8)
    constexpr bool UNPK = sizeof(TD) == 1;
    constexpr int RB = (UNPK ? 2 : 1) * PAIR_T;  // uint4 per buffer: [half][PAIR_T]
    uint4 *ring0 = smem;                         // slot 0
    uint4 *ring23 = smem + RB;                   // [row & 1][slot 2, 3]
    uint4 *ring1 = smem + 5 * RB;                // [row % 3]
    uint4 *stage = smem + 8 * RB;                // [PAIR_NBUF][NST][PAIR_T]
    const int NG = PAIR_T >> LOG2G, NI = NG - 2;
    const int tid = threadIdx.x;
    const int g = tid >> LOG2G, lane_g = tid & (G - 1);
    const int b = blockIdx.z;
    const int I0 = blockIdx.x * NI;
    const int Y0 = blockIdx.y * band, Y1 = min(Y0 + band, a.H);
    const uint32_t cA = a.colour, cB = a.colour ^ 1u;
    const bool lio = lane_g < a.nch;
    const int d0 = lane_g * CH;
    const uint32_t P = a.plane, Lp = (uint32_t)a.Lp, rowstep = (uint32_t)a.Wc * Lp;
    const uint8_t *Mr = a.M + (size_t)b * a.pairM;  // colour-B messages of iteration t-1
    uint8_t *Mw = a.Mw + (size_t)b * a.pairM;       // colour-B messages of iteration t+1
    const TD *Db = D + (size_t)b * a.pairD;

    uint32_t padm[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        padm[j] = !PAD ? 0u
                       : (d0 + j >= a.L ? (SIGNED ? 0x00007FFFu : 0x0000FFFFu) : 0u) |
                             (d0 + j + 8 >= a.L ? (SIGNED ? 0x7FFF0000u : 0xFFFF0000u) : 0u);

    // enqueue the global inputs of step `ya` (A row ya, B row ya-1) into stage[buf]
    // per-thread constants of the prefetch: the thread's colour-A index iA = I0-1+g and
    // colour-B index iA+1 in every row; offsets relative to the row's colour-A chunk
    const int iA = I0 - 1 + g;
    const bool colA = iA >= 0 && lio, colB = g < NI && iA + 1 < a.Wc && lio;
    const uint32_t rA0 = (uint32_t)iA * Lp + (uint32_t)d0;  // + ya * rowstep
    const uint8_t *MoB = Mr + (size_t)(cB * 4u) * P;        // colour-B planes of iteration t-1
    const TD *DA = Db + cA * P, *DB = Db + cB * P;

    // MODE 2: the parent columns iA - 1, iA, iA + 1 of the thread (chunk offsets,
    // parities, and whether the parent sends right (px < Wp - 1) / left (px > 0))
    const uint8_t *Mpb = MODEA == 2 ? a.Mp + (size_t)b * a.pairMp : nullptr;
    uint32_t pcol0 = 0, pcol1 = 0, pcol2 = 0, ppar0 = 0, ppar1 = 0, ppar2 = 0;
    bool pr0 = false, pr1 = false, pl1 = false, pl2 = false;
    if (MODEA == 2) {
        const int p0 = iA - 1, p1 = iA, p2 = iA + 1;
        pcol0 = (uint32_t)(p0 >> 1) * Lp + (uint32_t)d0;  // only used when p0 >= 0
        pcol1 = (uint32_t)(p1 >> 1) * Lp + (uint32_t)d0;
        pcol2 = (uint32_t)(p2 >> 1) * Lp + (uint32_t)d0;
        ppar0 = (uint32_t)p0 & 1u, ppar1 = (uint32_t)p1 & 1u, ppar2 = (uint32_t)p2 & 1u;
        pr0 = p0 < a.Wp - 1, pr1 = p1 < a.Wp - 1, pl1 = p1 > 0, pl2 = p2 > 0;
    }

    // enqueue the global inputs of step `ya` (A row ya, B row ya-1) into stage[buf]
    auto issue = [&](int ya, int buf) {
        uint4 *st = stage + (size_t)buf * NST * PAIR_T + tid;
        const uint32_t o = (cA + (uint32_t)ya) & 1u;  // colour-A parity of row ya (= colour B's of row ya-1)
        const int xA = 2 * iA + (int)o;
        const bool okA = colA && (unsigned)ya < (unsigned)a.H && xA < a.W;
        const uint32_t rA = rA0 + (uint32_t)ya * rowstep;
        if (MODEA == 0) {
            const bool v0 = okA && ya > 0, v1 = okA && ya < a.H - 1, v2 = okA && xA > 0, v3 = okA && xA < a.W - 1;
            cp_async16(st + 0 * PAIR_T, MoB + (v0 ? P + rA - rowstep : 0u), v0);
            cp_async16(st + 1 * PAIR_T, MoB + (v1 ? rA + rowstep : 0u), v1);
            cp_async16(st + 2 * PAIR_T, MoB + (v2 ? 3u * P + rA + (o - 1u) * Lp : 0u), v2);
            cp_async16(st + 3 * PAIR_T, MoB + (v3 ? 2u * P + rA + o * Lp : 0u), v3);
        } else if (MODEA == 2) {
            // the parent of (xA, y) is (xA >> 1, y >> 1) = (iA, y >> 1): the vertical
            // neighbours' parents sit in column iA, the left / right ones' in columns
            // iA - 1 + o / iA + o (per-thread constants pcol / ppar / pr / pl, above);
            // neighbour k's parent sends on slot k ^ 1
            const int Y = ya >> 1, pyu = (ya - 1) >> 1, pyd = (ya + 1) >> 1;
            const uint32_t rowp = (uint32_t)a.Wcp * Lp, PP = a.planep;
            const uint32_t cm = o ? pcol1 : pcol0, cq = o ? pcol2 : pcol1;  // left / right parents' columns
            const uint32_t pm = o ? ppar1 : ppar0, pq = o ? ppar2 : ppar1;  // and parities
            const bool v0 = okA && ya > 0 && pyu < a.Hp - 1;                  // up: the parent's slot 1
            const bool v1 = okA && ya < a.H - 1 && pyd > 0;                   // down: slot 0
            const bool v2 = okA && xA > 0 && (o ? pr1 : pr0);                 // left: slot 3 (px < Wp - 1)
            const bool v3 = okA && xA < a.W - 1 && (o ? pl2 : pl1);           // right: slot 2 (px > 0)
            const uint32_t o0 = v0 ? (((ppar1 + (uint32_t)pyu) & 1u) * 4u + 1u) * PP + (uint32_t)pyu * rowp + pcol1 : 0u;
            const uint32_t o1 = v1 ? (((ppar1 + (uint32_t)pyd) & 1u) * 4u) * PP + (uint32_t)pyd * rowp + pcol1 : 0u;
            const uint32_t o2 = v2 ? (((pm + (uint32_t)Y) & 1u) * 4u + 3u) * PP + (uint32_t)Y * rowp + cm : 0u;
            const uint32_t o3 = v3 ? (((pq + (uint32_t)Y) & 1u) * 4u + 2u) * PP + (uint32_t)Y * rowp + cq : 0u;
            cp_async16(st + 0 * PAIR_T, Mpb + o0, v0);
            cp_async16(st + 1 * PAIR_T, Mpb + o1, v1);
            cp_async16(st + 2 * PAIR_T, Mpb + o2, v2);
            cp_async16(st + 3 * PAIR_T, Mpb + o3, v3);
        }
        {
            const uint4 *dp = reinterpret_cast<const uint4 *>(DA + (okA ? rA : 0u));
#pragma unroll
            for (int w = 0; w < DW; ++w) cp_async16(st + (4 + w) * PAIR_T, dp + w, okA);
        }
        {
            // colour-B pixel iA+1 of row ya-1: x = xA + 2, chunk offset rA - rowstep + Lp
            const int yb = ya - 1;
            const bool okB = colB && yb >= Y0 && yb < Y1 && xA + 2 < a.W;
            const uint4 *dp = reinterpret_cast<const uint4 *>(DB + (okB ? rA - rowstep + Lp : 0u));
#pragma unroll
            for (int w = 0; w < DW; ++w) cp_async16(st + (4 + DW + w) * PAIR_T, dp + w, okB);
        }
        cp_async_commit();
    };

    issue(Y0 - 1, 0);
    int s = 0;
#pragma unroll 1
    for (int ya = Y0 - 1; ya <= Y1; ++ya, ++s) {
        cp_async_wait_all();  // this step's inputs (this thread's own copies)
        const uint4 *st = stage + (size_t)(PAIR_NBUF == 2 ? (s & 1) : 0) * NST * PAIR_T + tid;
        uint4 sv[NST];  // NBUF 1: the step's staged inputs, moved to registers before the refill
        if (PAIR_NBUF == 1) {
#pragma unroll
            for (int k = 0; k < NST; ++k) sv[k] = st[k * PAIR_T];
            st = sv;
        }
        if (ya + 1 <= Y1) issue(ya + 1, PAIR_NBUF == 2 ? (s + 1) & 1 : 0);
        constexpr int SS = PAIR_NBUF == 2 ? PAIR_T : 1;  // stride between staged chunks
        // ---- A-phase: colour-A pixel index I0-1+g of row ya (incl. the halo pixels)
        if (ya >= 0 && ya < a.H) {
            uint32_t dv[8], in[4][8];
#pragma unroll
            for (int k = 0; k < 4; ++k) unpack_u8(MODEA == 1 ? make_uint4(0u, 0u, 0u, 0u) : st[k * SS], in[k]);
            if (sizeof(TD) == 1) {
                unpack_u8(st[4 * SS], dv);
            } else {
                const uint4 lo = st[4 * SS], hi = st[5 * SS];
                dv[0] = lo.x, dv[1] = lo.y, dv[2] = lo.z, dv[3] = lo.w;
                dv[4] = hi.x, dv[5] = hi.y, dv[6] = hi.z, dv[7] = hi.w;
            }
            // (staged chunks of pixels outside the image are zero)
            if (FIN) {  // a5 for the colour-A pixel: D + its 4 incoming, ties -> smallest label
                const uint32_t lab = wta_key16<PAD>(dv, in, d0, a.L, G);
                const int xA = 2 * iA + (int)((cA + (uint32_t)ya) & 1u);
                if (lane_g == 0 && colA && xA < a.W && g >= 1 && g <= NI && ya >= Y0 && ya < Y1)
                    a.disp[((size_t)b * a.H + ya) * a.W + xA] = (int32_t)lab;
            }
            uint4 *const dst[4] = {ring0 + tid, ring1 + (size_t)((ya + 3) % 3) * RB + tid,
                                   ring23 + (size_t)((ya & 1) * 2 + 0) * RB + tid,
                                   ring23 + (size_t)((ya & 1) * 2 + 1) * RB + tid};
            outgoing<PAD, SIGNED, GT>(a, dv, in, padm, lane_g, [&](int k, const uint32_t o8[8]) {
                if (UNPK) {
                    dst[k][0] = make_uint4(o8[0], o8[1], o8[2], o8[3]);
                    dst[k][PAIR_T] = make_uint4(o8[4], o8[5], o8[6], o8[7]);
                } else {
                    dst[k][0] = pack_u8(o8);
                }
            });
        }
        __syncthreads();
        // ---- B-phase: colour-B pixel index I0+g of row yb = ya-1, from the ring
        const int yb = ya - 1;
        if (yb >= Y0 && yb < Y1) {  // block-uniform: every lane takes part in the group shuffles
            const uint32_t o = (cA + (uint32_t)ya) & 1u;  // colour-B parity of row yb
            const int x = 2 * (iA + 1) + (int)o;
            const bool io = colB && x < a.W;
            const bool has[4] = {yb > 0, yb < a.H - 1, x > 0, x < a.W - 1};
            const uint32_t r = rA0 + (uint32_t)yb * rowstep + Lp;
            // A(i, yb-1) sends down (slot 1), A(i, yb+1) up (slot 0), A(i-1+o, yb) right
            // (slot 3), A(i+o, yb) left (slot 2); the group of A index j is j - (I0 - 1)
            const uint4 *src[4] = {ring1 + (size_t)((yb + 2) % 3) * RB + (g + 1) * G + lane_g,
                                   ring0 + (g + 1) * G + lane_g,
                                   ring23 + (size_t)((yb & 1) * 2 + 1) * RB + (g + (int)o) * G + lane_g,
                                   ring23 + (size_t)((yb & 1) * 2 + 0) * RB + (g + 1 + (int)o) * G + lane_g};
            uint32_t dv[8], in[4][8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool v = io && has[k];
                if (UNPK) {
                    const uint4 lo = v ? src[k][0] : make_uint4(0u, 0u, 0u, 0u);
                    const uint4 hi = v ? src[k][PAIR_T] : make_uint4(0u, 0u, 0u, 0u);
                    in[k][0] = lo.x, in[k][1] = lo.y, in[k][2] = lo.z, in[k][3] = lo.w;
                    in[k][4] = hi.x, in[k][5] = hi.y, in[k][6] = hi.z, in[k][7] = hi.w;
                } else {
                    unpack_u8(v ? src[k][0] : make_uint4(0u, 0u, 0u, 0u), in[k]);
                }
            }
            if (sizeof(TD) == 1) {
                unpack_u8(st[(4 + DW) * SS], dv);
            } else {
                const uint4 lo = st[(4 + DW) * SS], hi = st[(5 + DW) * SS];
                dv[0] = lo.x, dv[1] = lo.y, dv[2] = lo.z, dv[3] = lo.w;
                dv[4] = hi.x, dv[5] = hi.y, dv[6] = hi.z, dv[7] = hi.w;
            }
            if (FIN) {  // a5 for the colour-B pixel from colour A's final messages
                const uint32_t lab = wta_key16<PAD>(dv, in, d0, a.L, G);
                if (lane_g == 0 && io) a.disp[((size_t)b * a.H + yb) * a.W + x] = (int32_t)lab;
                (void)r;
            } else {
                uint8_t *Mo = Mw + (size_t)(cB * 4u) * P + r;
                outgoing<PAD, SIGNED, GT>(a, dv, in, padm, lane_g, [&](int k, const uint32_t o8[8]) {
                    if (io) *reinterpret_cast<uint4 *>(Mo + (size_t)k * P) = pack_u8(o8);
                });
            }
        }
        __syncthreads();
    }
}

size_t pair_smem_bytes(int dbytes)
{
    const int DW = dbytes == 1 ? 1 : 2;
    return (size_t)(8 * (dbytes == 1 ? 2 : 1) + PAIR_NBUF * (4 + 2 * DW)) * PAIR_T * sizeof(uint4);
}

cudaError_t launch_update_pair(const void *D, int dbytes, const FastArgs &a, int B, int mode, bool sgn, int band,
                               cudaStream_t st, bool fin)
{
    const int NI = (PAIR_T >> a.log2G) - 2;
    dim3 grid((unsigned)((a.Wc + NI - 1) / NI), (unsigned)((a.H + band - 1) / band), (unsigned)B);
    const size_t smem = pair_smem_bytes(dbytes);
    const bool pad = (a.L % CH) != 0 || a.G != a.nch;
#define VSBP_KG(TD_, MODE_, PAD_, SG_, GT_)                                                                     \
    do {                                                                                                        \
        auto kf = k_update_pair<TD_, MODE_, PAD_, SG_, GT_, false>;                                             \
        static cudaError_t attr = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (attr != cudaSuccess) return attr;                                                                   \
        kf<<<grid, PAIR_T, smem, st>>>(a, (const TD_ *)D, band);                                                \
    } while (0)
    // the lane-group size is a compile-time constant for L = 64 (G = 4) and L = 128 (G = 8)
#define VSBP_K(TD_, MODE_, PAD_, SG_)                                   \
    do {                                                                \
        if (!PAD_ && a.G == 4) VSBP_KG(TD_, MODE_, PAD_, SG_, 4);       \
        else if (!PAD_ && a.G == 8) VSBP_KG(TD_, MODE_, PAD_, SG_, 8);  \
        else VSBP_KG(TD_, MODE_, PAD_, SG_, 0);                         \
    } while (0)
#define VSBP_S(TD_, MODE_, PAD_) \
    if (sgn) VSBP_K(TD_, MODE_, PAD_, true); else VSBP_K(TD_, MODE_, PAD_, false);
#define VSBP_P(TD_, MODE_) \
    if (pad) { VSBP_S(TD_, MODE_, true) } else { VSBP_S(TD_, MODE_, false) }
#define VSBP_M(TD_)              \
    switch (mode) {              \
    case 0: VSBP_P(TD_, 0) break; \
    case 1: VSBP_P(TD_, 1) break; \
    default: VSBP_P(TD_, 2) break; \
    }
    if (fin) {
        // the final iteration + WTA: u8 costs, MODE 0 only (use_final)
        if (dbytes != 1 || mode != 0) return cudaErrorInvalidValue;
#define VSBP_F(PAD_, SG_, GT_)                                                                                  \
    do {                                                                                                        \
        auto kf = k_update_pair<uint8_t, 0, PAD_, SG_, GT_, true>;                                              \
        static cudaError_t attr = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (attr != cudaSuccess) return attr;                                                                   \
        kf<<<grid, PAIR_T, smem, st>>>(a, (const uint8_t *)D, band);                                            \
    } while (0)
        if (!pad && a.G == 4) {
            if (sgn) VSBP_F(false, true, 4); else VSBP_F(false, false, 4);
        } else if (pad) {
            if (sgn) VSBP_F(true, true, 0); else VSBP_F(true, false, 0);
        } else {
            if (sgn) VSBP_F(false, true, 0); else VSBP_F(false, false, 0);
        }
#undef VSBP_F
    } else if (dbytes == 1) {
        VSBP_M(uint8_t)
    } else {
        VSBP_M(uint16_t)
    }
#undef VSBP_M
#undef VSBP_P
#undef VSBP_S
#undef VSBP_K
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_update_fast(const void *D, int dbytes, const FastArgs &a, int B, int mode, bool wta, bool sgn,
                               cudaStream_t st)
{
    const long threads = (long)a.npix * a.G;
    dim3 grid((unsigned)((threads + 255) / 256), (unsigned)B);
    const bool pad = (a.L % CH) != 0 || a.G != a.nch;
#define VSBP_K(TD_, MODE_, PAD_, WTA_, SG_) k_update_fast<TD_, MODE_, PAD_, WTA_, SG_><<<grid, 256, 0, st>>>(a, (const TD_ *)D)
#define VSBP_S(TD_, MODE_, PAD_, WTA_) \
    if (sgn) VSBP_K(TD_, MODE_, PAD_, WTA_, true); else VSBP_K(TD_, MODE_, PAD_, WTA_, false);
#define VSBP_W(TD_, MODE_, PAD_) \
    if (wta) { VSBP_S(TD_, MODE_, PAD_, true) } else { VSBP_S(TD_, MODE_, PAD_, false) }
#define VSBP_P(TD_, MODE_) \
    if (pad) { VSBP_W(TD_, MODE_, true) } else { VSBP_W(TD_, MODE_, false) }
#define VSBP_M(TD_)                                   \
    switch (mode) {                                   \
    case 0: VSBP_P(TD_, 0) break;                     \
    case 1: VSBP_P(TD_, 1) break;                     \
    case 2: VSBP_P(TD_, 2) break;                     \
    default:                                          \
        if (pad) VSBP_K(TD_, 3, true, true, false);   \
        else VSBP_K(TD_, 3, false, true, false);      \
        break;                                        \
    }
    if (dbytes == 0) {
        VSBP_M(ImgD)
    } else if (dbytes == 1) {
        VSBP_M(uint8_t)
    } else {
        VSBP_M(uint16_t)
    }
#undef VSBP_M
#undef VSBP_P
#undef VSBP_W
#undef VSBP_S
#undef VSBP_K
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
