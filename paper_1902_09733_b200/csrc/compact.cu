// compact.cu -- a8: the per-pair point cloud as a PACKED list of valid points in
// raster order ("a point cloud ... for each image pair"; SURVEY 8(a) a8
// "compacted xyz"), sm_100a.
//
// For B pairs of full-res disparity disp[B][H][W] (px) the valid pixels
// (d >= min_disp, R-21) are reprojected by Eq.3 (R-20; the same f32
// arithmetic as the fused JBU+reprojection kernel, so a packed point is
// bit-identical to the dense cloud's entry) and written to xyz[n][3] in
// (pair, row, column) order, with offsets[b] = index of pair b's first point and
// offsets[B] = the total.
//
// One pass, decoupled look-back (a single-pass prefix scan): the flattened
// (pair, pixel) range is cut into tiles of CC_TILE pixels that never straddle a
// pair boundary; a CTA takes the next tile from a ticket counter (so tiles start
// in order and the look-back cannot deadlock), counts its valid pixels, publishes
// that aggregate, then warp 0 walks back over its predecessors' descriptors
// (aggregate or inclusive prefix, 64-bit words: 2 status bits + 62-bit value)
// until an inclusive prefix closes the sum, and publishes its own inclusive
// prefix.  The tile's points are packed in shared memory and stored as one
// contiguous coalesced run.  HBM traffic: 4 B read per pixel + 12 B written per
// valid point (+ 8 B of descriptor per tile).
#include <cstdint>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

constexpr int CC_T = 256;                // threads per CTA
constexpr int CC_E = 8;                  // pixels per thread (the tile's packed points fit 24 KB of smem)
constexpr int CC_TILE = CC_T * CC_E;     // pixels per tile
constexpr unsigned long long CC_FLAG_A = 1ull << 62, CC_FLAG_P = 2ull << 62, CC_VAL = (1ull << 62) - 1;

struct CompactArgs {
    float q[16];
    float min_disp;
    int W, HW, tiles_per_pair, B;
    long long cap;                       // capacity of xyz in points
};

__device__ __forceinline__ float cc_rcp(float d)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    return r;
}

__device__ __forceinline__ unsigned long long ld_desc(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_desc(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <bool VEC>
__global__ void __launch_bounds__(CC_T) k_compact(const float *__restrict__ disp, const __grid_constant__ CompactArgs a,
                                                  float *__restrict__ xyz, long long *__restrict__ offsets,
                                                  unsigned long long *__restrict__ n_valid,
                                                  unsigned long long *__restrict__ desc, unsigned *__restrict__ ticket)
{
    __shared__ float sOut[CC_TILE * 3];
    __shared__ int sWarp[CC_T / 32];
    __shared__ int sTile;
    __shared__ long long sExcl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) sTile = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int t = sTile;
    const int b = t / a.tiles_per_pair;
    const int p0 = (t - b * a.tiles_per_pair) * CC_TILE;    // first pixel of the tile inside pair b
    const int n = min(CC_TILE, a.HW - p0);
    const float *src = disp + (size_t)b * a.HW + p0;

    // ---- load this thread's CC_E consecutive pixels, flag the valid ones
    float d[CC_E];
    const int i0 = tid * CC_E;
    if (VEC && i0 + CC_E <= n) {
        const float4 *s4 = reinterpret_cast<const float4 *>(src + i0);
#pragma unroll
        for (int j = 0; j < CC_E / 4; ++j) {
            const float4 v = __ldcs(s4 + j);
            d[4 * j] = v.x;
            d[4 * j + 1] = v.y;
            d[4 * j + 2] = v.z;
            d[4 * j + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < CC_E; ++j) d[j] = i0 + j < n ? src[i0 + j] : 0.f;
    }
    unsigned valid = 0;
#pragma unroll
    for (int j = 0; j < CC_E; ++j)
        if (i0 + j < n && d[j] >= a.min_disp) valid |= 1u << j;
    const int cnt = __popc(valid);

    // ---- block exclusive scan of the per-thread counts
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) sWarp[warp] = incl;
    __syncthreads();
    int wbase = 0, total = 0;
#pragma unroll
    for (int w = 0; w < CC_T / 32; ++w) {
        const int v = sWarp[w];
        wbase += w < warp ? v : 0;
        total += v;
    }
    const int texcl = wbase + incl - cnt;

    // ---- decoupled look-back over the preceding tiles (warp 0)
    if (warp == 0) {
        if (t == 0) {
            if (lane == 0) {
                st_desc(desc, CC_FLAG_P | (unsigned long long)total);
                sExcl = 0;
            }
        } else {
            if (lane == 0) st_desc(desc + t, CC_FLAG_A | (unsigned long long)total);
            long long excl = 0;
            int pos = t - 1;
            while (true) {
                const int idx = pos - lane;
                unsigned long long v = idx >= 0 ? ld_desc(desc + idx) : CC_FLAG_P;
                if (__any_sync(FULL, (v >> 62) == 0)) continue;  // a predecessor has not published yet
                const unsigned isP = __ballot_sync(FULL, (v >> 62) == 2);
                const int firstP = isP ? __ffs(isP) - 1 : 32;    // nearest inclusive prefix
                long long part = lane <= firstP ? (long long)(v & CC_VAL) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
                excl += part;
                if (isP) break;
                pos -= 32;
            }
            if (lane == 0) {
                st_desc(desc + t, CC_FLAG_P | (unsigned long long)(excl + total));
                sExcl = excl;
            }
        }
    }

    // ---- Eq.3 for the valid pixels, packed into shared memory (overlaps the look-back)
    int v = (p0 + i0) / a.W;
    int u = p0 + i0 - v * a.W;
    int k = texcl;
#pragma unroll
    for (int j = 0; j < CC_E; ++j, ++u) {
        while (u >= a.W) {
            u -= a.W;
            ++v;
        }
        if (!(valid >> j & 1)) continue;
        const float fu = (float)u, fv = (float)v;
        float h[4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
            h[r] = fmaf(a.q[4 * r + 2], d[j], fmaf(a.q[4 * r], fu, fmaf(a.q[4 * r + 1], fv, a.q[4 * r + 3])));
        const float rW = cc_rcp(h[3]);
        sOut[3 * k] = h[0] * rW;
        sOut[3 * k + 1] = h[1] * rW;
        sOut[3 * k + 2] = h[2] * rW;
        ++k;
    }
    __syncthreads();

    // ---- one contiguous, coalesced store of the tile's 3 * total floats
    const long long base = sExcl;
    const long long lim = min((long long)total, a.cap - base);  // points beyond the capacity are dropped
    float *dst = xyz + 3 * base;
    for (int e = tid; e < 3 * lim; e += CC_T) __stcs(dst + e, sOut[e]);
    if (tid == 0) {
        if (p0 == 0) offsets[b] = base;
        if (t == a.B * a.tiles_per_pair - 1) offsets[a.B] = base + total;
        if (total) atomicAdd(n_valid + b, (unsigned long long)total);
    }
}

size_t compact_workspace_bytes(int B, int W, int H)
{
    const long long tiles = (long long)B * (((long long)W * H + CC_TILE - 1) / CC_TILE);
    return (size_t)(tiles * 8 + 256);
}

cudaError_t launch_compact(int B, const float *disp, int W, int H, const float Qf[16], float min_disp, float *xyz,
                           long long cap, long long *offsets, unsigned long long *n_valid, void *ws,
                           cudaStream_t st)
{
    CompactArgs a;
    for (int i = 0; i < 16; ++i) a.q[i] = Qf[i];
    a.min_disp = min_disp;
    a.W = W;
    a.HW = W * H;
    a.tiles_per_pair = (a.HW + CC_TILE - 1) / CC_TILE;
    a.B = B;
    a.cap = cap;
    const long long tiles = (long long)B * a.tiles_per_pair;
    unsigned *ticket = reinterpret_cast<unsigned *>(ws);
    unsigned long long *desc = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(ws) + 256);
    cudaError_t e = cudaMemsetAsync(ws, 0, (size_t)tiles * 8 + 256, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(n_valid, 0, sizeof(unsigned long long) * (size_t)B, st);
    if (e != cudaSuccess) return e;
    const bool vec = (a.HW % 4 == 0) && (((uintptr_t)disp & 15) == 0);
    if (vec)
        k_compact<true><<<(unsigned)tiles, CC_T, 0, st>>>(disp, a, xyz, offsets, n_valid, desc, ticket);
    else
        k_compact<false><<<(unsigned)tiles, CC_T, 0, st>>>(disp, a, xyz, offsets, n_valid, desc, ticket);
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
