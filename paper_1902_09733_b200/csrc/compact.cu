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
// Three short kernels, no inter-CTA waiting: every row of every pair is cut into
// SEGMENTS of CC_SEG = 128 consecutive pixels (the last one of a row shorter), so the
// segments in (pair, row, segment) order are the pixels in raster order;
//   k_compact_count  counts each segment's valid pixels, one warp per segment (skipped
//                    when the JBU kernel has already counted them while producing
//                    disp -- jbu_compact_batch: one warp row of the JBU is one segment,
//                    the a6 kernel is EX2-bound, counting is free);
//   k_compact_chunk / k_compact_scan  exclusive prefix of the segment counts -> each
//                    segment's first output index, offsets[B+1] and n_valid[B];
//   k_compact_write  one warp per segment: 4 coalesced loads per lane, ballots give
//                    each valid pixel its rank inside the segment, Eq.3 in registers,
//                    the points stored at their packed index (the warp's stores cover
//                    one contiguous run).
// HBM traffic: 4 B read per pixel (8 B with the count pass) + 12 B written per valid
// point.  (Round 2 built 2048-pixel tiles first -- per-tile block scans, shared-memory
// staging, two atomics per JBU warp row -- and a single-pass decoupled look-back before
// that: DESIGN §12.)
#include <cstdint>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

constexpr int CC_T = 256;                // threads per CTA (8 warps)
constexpr int CC_SEG = 128;              // pixels per segment: one warp, 4 per lane
#ifndef VSBP_CC_WS
#define VSBP_CC_WS 4
#endif
constexpr int CC_WS = VSBP_CC_WS;        // segments per warp in the write kernel
struct CompactArgs {
    float q[16];
    float min_disp;
    int W, HW, segs, tiles_per_pair, B;  // segs = segments per row, tiles_per_pair = H * segs
    long long cap;                       // capacity of xyz in points
};

__device__ __forceinline__ float cc_rcp(float d)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    return r;
}

// segment t -> (pair b, index tl inside the pair, first pixel p0 inside the pair,
// pixel count n)
__device__ __forceinline__ void seg_of(const CompactArgs &a, int t, int &b, int &tl, int &p0, int &n)
{
    b = t / a.tiles_per_pair;
    tl = t - b * a.tiles_per_pair;
    const int y = tl / a.segs, x0 = (tl - y * a.segs) * CC_SEG;
    p0 = y * a.W + x0;
    n = min(CC_SEG, a.W - x0);
}

__global__ void __launch_bounds__(CC_T) k_compact_count(const float *__restrict__ disp, const CompactArgs a, int tiles,
                                                        int *__restrict__ tile_cnt)
{
    const int t = blockIdx.x * (CC_T / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (t >= tiles) return;
    int b, tl, p0, n;
    seg_of(a, t, b, tl, p0, n);
    const float *src = disp + (size_t)b * a.HW + p0;
    int c = 0;
#pragma unroll
    for (int k = 0; k < CC_SEG / 32; ++k) {
        const int e = 32 * k + lane;
        c += (e < n && __ldcs(src + e) >= a.min_disp) ? 1 : 0;
    }
    c = __reduce_add_sync(FULL, c);
    if (lane == 0) tile_cnt[t] = c;
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
    // this chunk's base: the sum of the earlier chunks' totals, summed by the whole
    // block (hundreds of chunks at the bench's 4.3 M segments)
    long long part = 0;
    for (int c = threadIdx.x; c < (int)blockIdx.x; c += CS_T) part += chunk_sum[c];
    long long base;
    block_excl_scan(part, sW, base);
    __syncthreads();  // sW is reused below
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

// One warp per segment (CC_WS segments per warp): lane l loads pixels l, l+32, l+64,
// l+96 of its segment (coalesced), so the raster order inside the segment is
// (k, lane) and a valid pixel's rank is the popcounts of the earlier ballots plus the
// lanes below it in its own.  The valid points of one k land at consecutive indices:
// each store instruction covers one contiguous run.
__global__ void __launch_bounds__(CC_T) k_compact_write(const float *__restrict__ disp, const __grid_constant__ CompactArgs a,
                                                        int tiles, const long long *__restrict__ tile_off,
                                                        float *__restrict__ xyz, const long long *__restrict__ offsets,
                                                        unsigned long long *__restrict__ n_valid)
{
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int w = blockIdx.x * (CC_T / 32) + (threadIdx.x >> 5);
#pragma unroll 1
    for (int i = 0; i < CC_WS; ++i) {
        const int t = w * CC_WS + i;
        if (t >= tiles) return;
        int b, tl, p0, n;
        seg_of(a, t, b, tl, p0, n);
        if (tl == 0 && lane == 0) n_valid[b] = (unsigned long long)(offsets[b + 1] - offsets[b]);
        const float *src = disp + (size_t)b * a.HW + p0;
        float d[CC_SEG / 32];
        unsigned ball[CC_SEG / 32];
#pragma unroll
        for (int k = 0; k < CC_SEG / 32; ++k) {
            const int e = 32 * k + lane;
            d[k] = e < n ? __ldcs(src + e) : 0.f;
            ball[k] = __ballot_sync(FULL, e < n && d[k] >= a.min_disp);
        }
        const long long base = tile_off[t];
        const int y = p0 / a.W, x0 = p0 - y * a.W;
        const float fv = (float)y;
        int r = 0;
#pragma unroll
        for (int k = 0; k < CC_SEG / 32; ++k) {
            if (ball[k] >> lane & 1) {
                const long long idx = base + r + __popc(ball[k] & lt);
                const float fu = (float)(x0 + 32 * k + lane);
                float h[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    h[q] = fmaf(a.q[4 * q + 2], d[k], fmaf(a.q[4 * q], fu, fmaf(a.q[4 * q + 1], fv, a.q[4 * q + 3])));
                const float rW = cc_rcp(h[3]);
                if (idx < a.cap) {  // points beyond the capacity are dropped
                    float *o = xyz + 3 * idx;
                    __stcs(o, h[0] * rW);
                    __stcs(o + 1, h[1] * rW);
                    __stcs(o + 2, h[2] * rW);
                }
            }
            r += __popc(ball[k]);
        }
    }
}

int compact_segs_per_row(int W) { return (W + CC_SEG - 1) / CC_SEG; }
int compact_tiles_per_pair(int W, int H) { return H * compact_segs_per_row(W); }

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
    a.segs = compact_segs_per_row(W);
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
    const long long wpc = (long long)(CC_T / 32) * CC_WS;  // segments per CTA
    k_compact_write<<<(unsigned)((tiles + wpc - 1) / wpc), CC_T, 0, st>>>(disp, a, (int)tiles, toff, xyz, offsets,
                                                                          n_valid);
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
    k_compact_count<<<(unsigned)((tiles + CC_T / 32 - 1) / (CC_T / 32)), CC_T, 0, st>>>(disp, a, (int)tiles,
                                                                                       compact_counts(ws));
    note_launch();
    return launch_compact_from_counts(B, disp, W, H, Qf, min_disp, xyz, cap, offsets, n_valid, ws, st);
}

}  // namespace vsbp
