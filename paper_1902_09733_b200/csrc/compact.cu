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
// Three short kernels, no inter-CTA waiting: the flattened (pair, pixel) range is
// cut into tiles of CC_TILE consecutive pixels that never straddle a pair boundary;
//   k_compact_count  counts each tile's valid pixels (skipped when the JBU kernel
//                    has already accumulated the counts while producing disp --
//                    jbu_compact_batch: the a6 kernel is EX2-bound, counting is free);
//   k_compact_scan   one CTA: exclusive prefix of the tile counts -> each tile's
//                    first output index, offsets[B+1] and n_valid[B];
//   k_compact_write  re-derives each tile's in-tile ranks (ballots, round-strided
//                    pixel ownership), evaluates Eq.3 for its valid pixels into
//                    shared memory and stores the tile's points as one contiguous
//                    coalesced run.
// HBM traffic: 4 B read per pixel (8 B with the count pass) + 12 B written per valid
// point.  (A single-pass decoupled look-back was built first and measured slower:
// 2.8-4.3 ms per 128-pair launch, CTAs stalled at the barrier behind warp 0's
// look-back.)
#include <cstdint>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

constexpr int CC_T = 256;                // threads per CTA
constexpr int CC_E = 8;                  // pixels per thread (the tile's packed points fit 24 KB of smem)
constexpr int CC_TILE = CC_T * CC_E;     // pixels per tile
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

// tile t -> (pair b, first pixel p0 inside the pair, pixel count n)
__device__ __forceinline__ void tile_of(const CompactArgs &a, int t, int &b, int &p0, int &n)
{
    b = t / a.tiles_per_pair;
    p0 = (t - b * a.tiles_per_pair) * CC_TILE;
    n = min(CC_TILE, a.HW - p0);
}

__global__ void __launch_bounds__(CC_T) k_compact_count(const float *__restrict__ disp, const CompactArgs a,
                                                        int *__restrict__ tile_cnt)
{
    int b, p0, n;
    tile_of(a, blockIdx.x, b, p0, n);
    const float *src = disp + (size_t)b * a.HW + p0;
    int c = 0;
#pragma unroll
    for (int i = 0; i < CC_E; ++i) {
        const int e = i * CC_T + threadIdx.x;
        c += (e < n && __ldcs(src + e) >= a.min_disp) ? 1 : 0;
    }
    c = __reduce_add_sync(FULL, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(tile_cnt + blockIdx.x, c);
}

// The tile-count scan in two short kernels over chunks of CS_CHUNK tiles (a few
// dozen CTAs at the bench's 257K tiles): k_compact_chunk sums each chunk,
// k_compact_scan prefixes the chunk sums and block-scans its own chunk.
constexpr int CS_T = 1024, CS_V = 8, CS_CHUNK = CS_T * CS_V;

__device__ __forceinline__ long long block_excl_scan(long long x, long long *sW, long long &total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) sW[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const long long w = sW[lane];
        long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long v = __shfl_up_sync(FULL, wi, o);
            if (lane >= o) wi += v;
        }
        sW[lane] = wi - w;
        if (lane == 31) sW[32] = wi;
    }
    __syncthreads();
    total = sW[32];
    return sW[warp] + incl - x;
}

__global__ void __launch_bounds__(CS_T) k_compact_chunk(const int *__restrict__ tile_cnt, int tiles,
                                                        long long *__restrict__ chunk_sum)
{
    __shared__ long long sW[33];
    const int t0 = blockIdx.x * CS_CHUNK + threadIdx.x * CS_V;
    long long c = 0;
#pragma unroll
    for (int j = 0; j < CS_V; ++j) c += t0 + j < tiles ? tile_cnt[t0 + j] : 0;
    long long total;
    block_excl_scan(c, sW, total);
    if (threadIdx.x == 0) chunk_sum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(CS_T) k_compact_scan(const int *__restrict__ tile_cnt, int tiles,
                                                       const long long *__restrict__ chunk_sum, const CompactArgs a,
                                                       long long *__restrict__ tile_off, long long *__restrict__ offsets)
{
    __shared__ long long sW[33];
    long long base = 0;
    for (int c = 0; c < (int)blockIdx.x; ++c) base += chunk_sum[c];  // a few dozen chunks
    const int t0 = blockIdx.x * CS_CHUNK + threadIdx.x * CS_V;
    int v[CS_V];
    long long c = 0;
#pragma unroll
    for (int j = 0; j < CS_V; ++j) {
        v[j] = t0 + j < tiles ? tile_cnt[t0 + j] : 0;
        c += v[j];
    }
    long long total;
    long long run = base + block_excl_scan(c, sW, total);
#pragma unroll
    for (int j = 0; j < CS_V; ++j) {
        const int t = t0 + j;
        if (t < tiles) {
            tile_off[t] = run;
            if (t % a.tiles_per_pair == 0) offsets[t / a.tiles_per_pair] = run;
            if (t == tiles - 1) offsets[a.B] = run + v[j];
        }
        run += v[j];
    }
}

// Round i of a tile covers its pixels [i*CC_T, (i+1)*CC_T): lane l of warp w owns
// pixel i*CC_T + 32w + l, so every load is one coalesced 128-byte line per warp and
// the points of a round land at consecutive shared-memory slots (stride 3 floats:
// no bank conflicts).  Raster order = (round, warp, lane) order.
__global__ void __launch_bounds__(CC_T) k_compact_write(const float *__restrict__ disp, const __grid_constant__ CompactArgs a,
                                                        const long long *__restrict__ tile_off, float *__restrict__ xyz,
                                                        const long long *__restrict__ offsets,
                                                        unsigned long long *__restrict__ n_valid)
{
    constexpr int NW = CC_T / 32;
    __shared__ float sOut[CC_TILE * 3];
    __shared__ int sPre[CC_E * NW + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t = blockIdx.x;
    int b, p0, n;
    tile_of(a, t, b, p0, n);
    const float *src = disp + (size_t)b * a.HW + p0;
    if (p0 == 0 && tid == 0) n_valid[b] = (unsigned long long)(offsets[b + 1] - offsets[b]);

    // ---- load: one pixel per thread and round; ballot the valid ones
    float d[CC_E];
    unsigned ball[CC_E];
#pragma unroll
    for (int i = 0; i < CC_E; ++i) {
        const int e = i * CC_T + tid;
        d[i] = e < n ? __ldcs(src + e) : 0.f;
        ball[i] = __ballot_sync(FULL, e < n && d[i] >= a.min_disp);
    }
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < CC_E; ++i) sPre[i * NW + warp] = __popc(ball[i]);
    }
    __syncthreads();
    // ---- exclusive scan of the CC_E x NW (round, warp) counts, in raster order (warp 0)
    if (warp == 0) {
        static_assert(CC_E * NW == 64, "two counts per lane");
        const int c0 = sPre[2 * lane], c1 = sPre[2 * lane + 1];
        int incl = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
        }
        const int excl = incl - c0 - c1;
        sPre[2 * lane] = excl;
        sPre[2 * lane + 1] = excl + c0;
        if (lane == 31) sPre[CC_E * NW] = incl;
    }
    __syncthreads();
    const int total = sPre[CC_E * NW];

    // ---- Eq.3 for the valid pixels into their packed slots
    int v = (p0 + tid) / a.W;
    int u = p0 + tid - v * a.W;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < CC_E; ++i) {
        if (ball[i] >> lane & 1) {
            const int k = sPre[i * NW + warp] + __popc(ball[i] & lt);
            const float fu = (float)u, fv = (float)v;
            float h[4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
                h[r] = fmaf(a.q[4 * r + 2], d[i], fmaf(a.q[4 * r], fu, fmaf(a.q[4 * r + 1], fv, a.q[4 * r + 3])));
            const float rW = cc_rcp(h[3]);
            sOut[3 * k] = h[0] * rW;
            sOut[3 * k + 1] = h[1] * rW;
            sOut[3 * k + 2] = h[2] * rW;
        }
        u += CC_T;
        while (u >= a.W) {
            u -= a.W;
            ++v;
        }
    }
    __syncthreads();

    // ---- one contiguous, coalesced store of the tile's 3 * total floats: 8-byte
    // stores (conflict-free LDS.64 from shared memory) after a one-float head that
    // aligns the destination
    const long long base = tile_off[t];
    const long long lim = min((long long)total, a.cap - base);  // points beyond the capacity are dropped
    float *dst = xyz + 3 * base;
    const int nf = lim > 0 ? (int)(3 * lim) : 0;
    const int head = min(nf, (int)(((uintptr_t)dst >> 2) & 1));
    if (tid < head) __stcs(dst, sOut[0]);
    const int n2 = (nf - head) >> 1;
    float2 *d2 = reinterpret_cast<float2 *>(dst + head);
    if (head) {
        for (int q = tid; q < n2; q += CC_T) __stcs(d2 + q, make_float2(sOut[1 + 2 * q], sOut[2 + 2 * q]));
    } else {
        const float2 *s2 = reinterpret_cast<const float2 *>(sOut);
        for (int q = tid; q < n2; q += CC_T) __stcs(d2 + q, s2[q]);
    }
    if (tid == 0 && head + 2 * n2 < nf) __stcs(dst + nf - 1, sOut[nf - 1]);
}

int compact_tiles_per_pair(int W, int H) { return (W * H + CC_TILE - 1) / CC_TILE; }
int compact_tile_pixels() { return CC_TILE; }

size_t compact_workspace_bytes(int B, int W, int H)
{
    const long long tiles = (long long)B * compact_tiles_per_pair(W, H);
    const long long chunks = (tiles + CS_CHUNK - 1) / CS_CHUNK;
    return (size_t)(tiles * 12 + chunks * 8 + 512);  // int32 counts | int64 tile offsets | int64 chunk sums
}

static CompactArgs make_args(int B, int W, int H, const float Qf[16], float min_disp, long long cap)
{
    CompactArgs a;
    for (int i = 0; i < 16; ++i) a.q[i] = Qf[i];
    a.min_disp = min_disp;
    a.W = W;
    a.HW = W * H;
    a.tiles_per_pair = compact_tiles_per_pair(W, H);
    a.B = B;
    a.cap = cap;
    return a;
}

// workspace: int32 tile counts at ws (zeroed by compact_zero_counts), int64 tile
// offsets after them
int *compact_counts(void *ws) { return reinterpret_cast<int *>(ws); }
static long long *compact_offsets(void *ws, long long tiles)
{
    return reinterpret_cast<long long *>(reinterpret_cast<char *>(ws) + ((tiles * 4 + 255) / 256) * 256);
}

cudaError_t compact_zero_counts(int B, int W, int H, void *ws, cudaStream_t st)
{
    const long long tiles = (long long)B * compact_tiles_per_pair(W, H);
    return cudaMemsetAsync(ws, 0, (size_t)tiles * 4, st);
}

cudaError_t launch_compact_from_counts(int B, const float *disp, int W, int H, const float Qf[16], float min_disp,
                                       float *xyz, long long cap, long long *offsets, unsigned long long *n_valid,
                                       void *ws, cudaStream_t st)
{
    const CompactArgs a = make_args(B, W, H, Qf, min_disp, cap);
    const long long tiles = (long long)B * a.tiles_per_pair;
    long long *toff = compact_offsets(ws, tiles);
    long long *csum = toff + tiles;
    const unsigned chunks = (unsigned)((tiles + CS_CHUNK - 1) / CS_CHUNK);
    k_compact_chunk<<<chunks, CS_T, 0, st>>>(compact_counts(ws), (int)tiles, csum);
    k_compact_scan<<<chunks, CS_T, 0, st>>>(compact_counts(ws), (int)tiles, csum, a, toff, offsets);
    k_compact_write<<<(unsigned)tiles, CC_T, 0, st>>>(disp, a, toff, xyz, offsets, n_valid);
    note_launch(3);
    return cudaGetLastError();
}

cudaError_t launch_compact(int B, const float *disp, int W, int H, const float Qf[16], float min_disp, float *xyz,
                           long long cap, long long *offsets, unsigned long long *n_valid, void *ws,
                           cudaStream_t st)
{
    const CompactArgs a = make_args(B, W, H, Qf, min_disp, cap);
    const long long tiles = (long long)B * a.tiles_per_pair;
    cudaError_t e = compact_zero_counts(B, W, H, ws, st);
    if (e != cudaSuccess) return e;
    k_compact_count<<<(unsigned)tiles, CC_T, 0, st>>>(disp, a, compact_counts(ws));
    note_launch();
    return launch_compact_from_counts(B, disp, W, H, Qf, min_disp, xyz, cap, offsets, n_valid, ws, st);
}

}  // namespace vsbp
