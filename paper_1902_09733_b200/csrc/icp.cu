// icp.cu -- row f4: point-to-point ICP on GPU ("CUDA accelerated Iterative
// Closest Point (ICP) [6] ... on the point clouds calculated from low-resolution
// disparity maps using Equation 3"; R-36), sm_100a.
//
// float64 throughout (B200 runs FP64 at half the FP32 rate; the pairing is a
// floating-point decision, so it is taken in the same precision and operation
// order as the oracle: p = ((R00 x + R01 y) + R02 z) + t0, d2 = (dx dx + dy dy) + dz dz,
// explicit _rn intrinsics, no contraction).
//   * compaction: valid (non-NaN) points in input order, every stride-th source;
//   * a uniform hash grid of the targets with cell = max_dist: a target within
//     max_dist of p lies in p's 3x3x3 cells, so the grid search returns the brute-
//     force nearest whenever it is kept (ties: smaller target index);
//   * per iteration (launched max_iter times, device-side `done` flag, no host
//     sync): pairing, two deterministic block reductions (centroids, then the
//     centred 3x3 correlation), and a one-thread rigid solve by Horn's quaternion
//     method (4x4 cyclic Jacobi) that composes the update onto T.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "vsbp_internal.cuh"
#include "vsbp_kernels.h"

namespace vsbp {

constexpr int IC_T = 256;
constexpr unsigned long long IC_EMPTY = ~0ull;

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ unsigned long long cell_key(long long cx, long long cy, long long cz)
{
    return ((unsigned long long)(cx + (1 << 20)) << 42) | ((unsigned long long)(cy + (1 << 20)) << 21) |
           (unsigned long long)(cz + (1 << 20));
}

__device__ __forceinline__ unsigned hash_slot(unsigned long long k, unsigned mask)
{
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    return (unsigned)k & mask;
}

// ---------------------------------------------------------------- compaction
__global__ void k_icp_count(const float *__restrict__ xyz, int n, int *__restrict__ blk)
{
    __shared__ int s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    const int i = blockIdx.x * IC_T + threadIdx.x;
    const bool v = i < n && !isnan(xyz[3 * i]) && !isnan(xyz[3 * i + 1]) && !isnan(xyz[3 * i + 2]);
    const unsigned m = __ballot_sync(FULL, v);
    if ((threadIdx.x & 31) == 0) atomicAdd(&s, __popc(m));
    __syncthreads();
    if (threadIdx.x == 0) blk[blockIdx.x] = s;
}

// exclusive scan of n ints in one block (n small: one entry per 256 points)
__global__ void k_icp_scan(int *__restrict__ v, int n, int *__restrict__ total)
{
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int x = i < n ? v[i] : 0;
        // inclusive warp scan then block scan through shared memory
        int s = x;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, s, o);
            if ((threadIdx.x & 31) >= o) s += y;
        }
        __shared__ int ws[32];
        if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x < 32) {
            int w = threadIdx.x < (int)(blockDim.x >> 5) ? ws[threadIdx.x] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, w, o);
                if (threadIdx.x >= o) w += y;
            }
            ws[threadIdx.x] = w;
        }
        __syncthreads();
        const int pre = (threadIdx.x >= 32 ? ws[(threadIdx.x >> 5) - 1] : 0) + s - x;
        if (i < n) v[i] = carry + pre;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += pre + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

// valid points in order; keep ranks r with r % stride == 0 (as double xyz)
__global__ void k_icp_compact(const float *__restrict__ xyz, int n, const int *__restrict__ blk, int stride,
                              double *__restrict__ out)
{
    __shared__ int wsum[IC_T / 32];
    const int i = blockIdx.x * IC_T + threadIdx.x;
    const bool v = i < n && !isnan(xyz[3 * i]) && !isnan(xyz[3 * i + 1]) && !isnan(xyz[3 * i + 2]);
    const unsigned m = __ballot_sync(FULL, v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) wsum[w] = __popc(m);
    __syncthreads();
    int off = blk[blockIdx.x];
    for (int q = 0; q < w; ++q) off += wsum[q];
    const int r = off + __popc(m & ((1u << lane) - 1u));
    if (v && r % stride == 0) {
        const int o = r / stride;
        out[3 * o] = xyz[3 * i];
        out[3 * o + 1] = xyz[3 * i + 1];
        out[3 * o + 2] = xyz[3 * i + 2];
    }
}

// ---------------------------------------------------------------- hash grid of the targets
struct IcpGrid {
    unsigned long long *keys;  // [HT]
    unsigned *count;           // [HT]
    unsigned *start;           // [HT] first entry of the cell in pts (atomic allocation)
    unsigned *cursor;          // [HT]
    unsigned *total;           // [1] allocation counter
    double4 *pts;              // [nt] {x, y, z, index bits} grouped by cell (contiguous per cell)
    unsigned mask;
    double inv_cell, cell;
};

// cell coordinates, clamped to the 21-bit key range (clamped points share border
// cells, so a neighbour within max_dist is still found -- only slower)
__device__ __forceinline__ void cell_of(const double *p, double inv, long long c[3])
{
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double f = floor(dmul(p[a], inv));
        c[a] = (long long)fmin(fmax(f, -1048574.0), 1048574.0);
    }
}

__global__ void k_icp_insert(const double *__restrict__ Q, const int *__restrict__ nt_p, IcpGrid g)
{
    const int nt = *nt_p;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nt; i += gridDim.x * blockDim.x) {
        long long c[3];
        cell_of(Q + 3 * i, g.inv_cell, c);
        const unsigned long long k = cell_key(c[0], c[1], c[2]);
        unsigned s = hash_slot(k, g.mask);
        while (true) {
            const unsigned long long prev = atomicCAS(g.keys + s, IC_EMPTY, k);
            if (prev == IC_EMPTY || prev == k) break;
            s = (s + 1) & g.mask;
        }
        atomicAdd(g.count + s, 1u);
    }
}

// cell storage: each occupied cell gets a contiguous range of pts.  The ranges are
// allocated with one atomic per cell, so their order in memory is arbitrary; the
// pairing is order-independent (nearest by (d2, index)), so results are not.
__global__ void k_icp_alloc(IcpGrid g)
{
    for (unsigned s = blockIdx.x * blockDim.x + threadIdx.x; s <= g.mask; s += gridDim.x * blockDim.x) {
        const unsigned c = g.count[s];
        if (c) g.start[s] = atomicAdd(g.total, c);
    }
}

__global__ void k_icp_scatter(const double *__restrict__ Q, const int *__restrict__ nt_p, IcpGrid g)
{
    const int nt = *nt_p;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nt; i += gridDim.x * blockDim.x) {
        long long c[3];
        cell_of(Q + 3 * i, g.inv_cell, c);
        const unsigned long long k = cell_key(c[0], c[1], c[2]);
        unsigned s = hash_slot(k, g.mask);
        while (g.keys[s] != k) s = (s + 1) & g.mask;
        g.pts[g.start[s] + atomicAdd(g.cursor + s, 1u)] =
            make_double4(Q[3 * i], Q[3 * i + 1], Q[3 * i + 2], __longlong_as_double((long long)i));
    }
}

// ---------------------------------------------------------------- state shared by the iteration kernels
struct IcpState {
    double T[12];          // [R|t] row-major
    double prev_rms, rms;
    double cen[6];         // source and target centroids of this iteration
    int iters, done, converged, npairs;
};

// Nearest target of each transformed source point, IC_G lanes per point (the lanes
// split each cell's points; (d2, index) is reduced over the group after every cell,
// so every lane prunes with the group's best).  The 27 cells around p are visited
// own cell first; a cell is skipped when its box is farther from p than the best
// distance so far (or than max_dist): every point stored in it is at least that far,
// so the nearest by (d2, index) is unchanged.  The box bound is reduced by a margin
// of 1e-7 cells (far above the rounding of floor(x / cell)) and the comparison is
// strict, so ties are never pruned.
constexpr int IC_G = 8;

__device__ __forceinline__ void better(double &best, int &bj, double d2, int j)
{
    if (d2 < best || (d2 == best && (unsigned)j < (unsigned)bj)) {
        best = d2;
        bj = j;
    }
}

__global__ void __launch_bounds__(IC_T) k_icp_pair(const double *__restrict__ S, const int *__restrict__ ns_p,
                                                    IcpGrid g, const IcpState *__restrict__ st, double max_d2,
                                                    int *__restrict__ match, double *__restrict__ dist2)
{
    if (st->done) return;
    const int ns = *ns_p;
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) / IC_G;
    const int lg = threadIdx.x & (IC_G - 1);
    if (i >= ns) return;  // whole groups exit together (IC_G divides the block)
    const unsigned gmask = (0xFFFFFFFFu >> (32 - IC_G)) << ((threadIdx.x & 31) & ~(IC_G - 1));
    const double *T = st->T;
    double p[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
        p[a] = dadd(dadd(dadd(dmul(T[4 * a], S[3 * i]), dmul(T[4 * a + 1], S[3 * i + 1])), dmul(T[4 * a + 2], S[3 * i + 2])),
                    T[4 * a + 3]);
    long long c[3];
    cell_of(p, g.inv_cell, c);
    // distance from p to the lower / upper face of its cell along each axis (>= 0)
    double lo[3], hi[3];
    bool prune = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double f = floor(p[a] * g.inv_cell);
        prune = prune && fabs(f) < 1048000.0;  // clamped cells: no geometry, visit all 27
        const double m = 1e-7 * g.cell;
        lo[a] = fmax(p[a] - (double)c[a] * g.cell - m, 0.0);
        hi[a] = fmax((double)(c[a] + 1) * g.cell - p[a] - m, 0.0);
    }
    double best = INFINITY;
    int bj = -1;  // as unsigned: larger than every index
    for (int n = 0; n < 27; ++n) {
        // n = 0 is the own cell, then the 26 neighbours
        const int e = n == 0 ? 13 : (n <= 13 ? n - 1 : n);
        const int dx = e % 3 - 1, dy = (e / 3) % 3 - 1, dz = e / 9 - 1;
        if (prune) {
            const double bx = dx < 0 ? lo[0] : (dx > 0 ? hi[0] : 0.0);
            const double by = dy < 0 ? lo[1] : (dy > 0 ? hi[1] : 0.0);
            const double bz = dz < 0 ? lo[2] : (dz > 0 ? hi[2] : 0.0);
            const double bd2 = bx * bx + by * by + bz * bz;
            if (bd2 > fmin(best, max_d2) * (1.0 + 1e-12)) continue;
        }
        const unsigned long long k = cell_key(c[0] + dx, c[1] + dy, c[2] + dz);
        unsigned s = hash_slot(k, g.mask);
        unsigned long long ks;
        while ((ks = g.keys[s]) != IC_EMPTY && ks != k) s = (s + 1) & g.mask;
        if (ks != k) continue;
        const unsigned b0 = g.start[s], b1 = b0 + g.count[s];
        for (unsigned e2 = b0 + lg; e2 < b1; e2 += IC_G) {
            const double4 q = g.pts[e2];
            const double ex = dsub(p[0], q.x), ey = dsub(p[1], q.y), ez = dsub(p[2], q.z);
            better(best, bj, dadd(dadd(dmul(ex, ex), dmul(ey, ey)), dmul(ez, ez)), (int)__double_as_longlong(q.w));
        }
#pragma unroll
        for (int o = IC_G / 2; o > 0; o >>= 1)
            better(best, bj, __shfl_xor_sync(gmask, best, o, IC_G), __shfl_xor_sync(gmask, bj, o, IC_G));
    }
    if (lg == 0) {
        const bool keep = bj >= 0 && best <= max_d2;
        match[i] = keep ? bj : -1;
        dist2[i] = keep ? best : 0.0;
    }
}

// block sums of K doubles in a fixed tree order (deterministic)
template <int K>
__device__ __forceinline__ void block_sum(double v[K], double *out)
{
    __shared__ double sh[IC_T / 32][K];
#pragma unroll
    for (int k = 0; k < K; ++k)
        for (int o = 16; o > 0; o >>= 1) v[k] = dadd(v[k], __shfl_xor_sync(FULL, v[k], o));
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) sh[threadIdx.x >> 5][k] = v[k];
    __syncthreads();
    if (threadIdx.x == 0)
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int w = 0; w < IC_T / 32; ++w) s = dadd(s, sh[w][k]);
            out[k] = s;
        }
}

// pass 1: count, sum p (3), sum q (3), sum d2
__global__ void __launch_bounds__(IC_T) k_icp_sum1(const double *__restrict__ S, const int *__restrict__ ns_p,
                                                    const double *__restrict__ Q, const IcpState *__restrict__ st,
                                                    const int *__restrict__ match, const double *__restrict__ dist2,
                                                    double *__restrict__ part)
{
    if (st->done) return;
    const int ns = *ns_p;
    const double *T = st->T;
    double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = blockIdx.x * IC_T + threadIdx.x; i < ns; i += gridDim.x * IC_T) {
        const int j = match[i];
        if (j < 0) continue;
        v[0] = dadd(v[0], 1.0);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double pa = dadd(dadd(dadd(dmul(T[4 * a], S[3 * i]), dmul(T[4 * a + 1], S[3 * i + 1])),
                                        dmul(T[4 * a + 2], S[3 * i + 2])),
                                   T[4 * a + 3]);
            v[1 + a] = dadd(v[1 + a], pa);
            v[4 + a] = dadd(v[4 + a], Q[3 * j + a]);
        }
        v[7] = dadd(v[7], dist2[i]);
    }
    block_sum<8>(v, part + (size_t)blockIdx.x * 8);
}

__global__ void __launch_bounds__(IC_T) k_icp_centroid(const double *__restrict__ part, int nb, IcpState *st)
{
    if (st->done) return;
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = 0.0;
    for (int b = threadIdx.x; b < nb; b += IC_T)
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = dadd(v[k], part[(size_t)b * 8 + k]);
    __shared__ double tot[8];
    block_sum<8>(v, tot);
    __syncthreads();
    if (threadIdx.x == 0) {
        const double n = tot[0];
        st->npairs = (int)n;
        if (n == 0.0) {
            st->done = 1;
            st->iters = -1;
            st->converged = 0;
            st->rms = NAN;
            return;
        }
        for (int k = 0; k < 6; ++k) st->cen[k] = tot[1 + k] / n;
        st->rms = sqrt(tot[7] / n);
    }
}

// pass 2: the centred correlation H_ab = sum (p_a - pbar_a)(q_b - qbar_b)
__global__ void __launch_bounds__(IC_T) k_icp_sum2(const double *__restrict__ S, const int *__restrict__ ns_p,
                                                    const double *__restrict__ Q, const IcpState *__restrict__ st,
                                                    const int *__restrict__ match, double *__restrict__ part)
{
    if (st->done) return;
    const int ns = *ns_p;
    const double *T = st->T;
    double v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = 0.0;
    for (int i = blockIdx.x * IC_T + threadIdx.x; i < ns; i += gridDim.x * IC_T) {
        const int j = match[i];
        if (j < 0) continue;
        double pc[3], qc[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double pa = dadd(dadd(dadd(dmul(T[4 * a], S[3 * i]), dmul(T[4 * a + 1], S[3 * i + 1])),
                                        dmul(T[4 * a + 2], S[3 * i + 2])),
                                   T[4 * a + 3]);
            pc[a] = dsub(pa, st->cen[a]);
            qc[a] = dsub(Q[3 * j + a], st->cen[3 + a]);
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int c = 0; c < 3; ++c) v[3 * a + c] = dadd(v[3 * a + c], dmul(pc[a], qc[c]));
    }
    block_sum<9>(v, part + (size_t)blockIdx.x * 9);
}

// Horn's closed form: the unit quaternion maximising q^T N q is the eigenvector of
// the largest eigenvalue of the symmetric 4x4 N built from H (cyclic Jacobi).
__device__ void horn_rotation(const double H[9], double R[9])
{
    const double Sxx = H[0], Sxy = H[1], Sxz = H[2], Syx = H[3], Syy = H[4], Syz = H[5], Szx = H[6], Szy = H[7],
                 Szz = H[8];
    double N[4][4] = {{Sxx + Syy + Szz, Syz - Szy, Szx - Sxz, Sxy - Syx},
                      {Syz - Szy, Sxx - Syy - Szz, Sxy + Syx, Szx + Sxz},
                      {Szx - Sxz, Sxy + Syx, -Sxx + Syy - Szz, Syz + Szy},
                      {Sxy - Syx, Szx + Sxz, Syz + Szy, -Sxx - Syy + Szz}};
    double V[4][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, 1}};
    // fully unrolled so N and V stay in registers (a local-memory version took
    // ~150 us per solve); stop when the off-diagonal mass is negligible
    double diag = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) diag += N[i][i] * N[i][i];
    for (int sweep = 0; sweep < 50; ++sweep) {
        double off = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = i + 1; j < 4; ++j) off += N[i][j] * N[i][j];
        if (off <= 1e-40 * diag) break;
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = p + 1; q < 4; ++q) {
                if (N[p][q] == 0.0) continue;
                const double theta = (N[q][q] - N[p][p]) / (2.0 * N[p][q]);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll
                for (int k = 0; k < 4; ++k) {  // columns p, q of N
                    const double a = N[k][p], b = N[k][q];
                    N[k][p] = c * a - s * b;
                    N[k][q] = s * a + c * b;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {  // rows p, q
                    const double a = N[p][k], b = N[q][k];
                    N[p][k] = c * a - s * b;
                    N[q][k] = s * a + c * b;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double a = V[k][p], b = V[k][q];
                    V[k][p] = c * a - s * b;
                    V[k][q] = s * a + c * b;
                }
            }
    }
    // eigenvector of the largest eigenvalue (register selects, no dynamic indexing)
    double w = V[0][0], x = V[1][0], y = V[2][0], z = V[3][0], lm = N[0][0];
#pragma unroll
    for (int i = 1; i < 4; ++i)
        if (N[i][i] > lm) {
            lm = N[i][i];
            w = V[0][i], x = V[1][i], y = V[2][i], z = V[3][i];
        }
    const double nrm = sqrt(w * w + x * x + y * y + z * z);
    w /= nrm, x /= nrm, y /= nrm, z /= nrm;
    R[0] = w * w + x * x - y * y - z * z;
    R[1] = 2 * (x * y - w * z);
    R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);
    R[4] = w * w - x * x + y * y - z * z;
    R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);
    R[7] = 2 * (y * z + w * x);
    R[8] = w * w - x * x - y * y + z * z;
}

__global__ void __launch_bounds__(IC_T) k_icp_solve(const double *__restrict__ part, int nb, IcpState *st, int it,
                                                     double eps)
{
    if (st->done) return;
    double v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = 0.0;
    for (int b = threadIdx.x; b < nb; b += IC_T)
#pragma unroll
        for (int k = 0; k < 9; ++k) v[k] = dadd(v[k], part[(size_t)b * 9 + k]);
    __shared__ double Hs[9];
    block_sum<9>(v, Hs);
    __syncthreads();
    if (threadIdx.x != 0) return;
    double Rd[9];
    horn_rotation(Hs, Rd);
    double td[3];
    for (int a = 0; a < 3; ++a)
        td[a] = st->cen[3 + a] - (Rd[3 * a] * st->cen[0] + Rd[3 * a + 1] * st->cen[1] + Rd[3 * a + 2] * st->cen[2]);
    double Tn[12];
    for (int a = 0; a < 3; ++a) {
        for (int c = 0; c < 3; ++c)
            Tn[4 * a + c] = Rd[3 * a] * st->T[c] + Rd[3 * a + 1] * st->T[4 + c] + Rd[3 * a + 2] * st->T[8 + c];
        Tn[4 * a + 3] = Rd[3 * a] * st->T[3] + Rd[3 * a + 1] * st->T[7] + Rd[3 * a + 2] * st->T[11] + td[a];
    }
    for (int k = 0; k < 12; ++k) st->T[k] = Tn[k];
    st->iters = it;
    if (fabs(st->rms - st->prev_rms) < eps) {
        st->done = 1;
        st->converged = 1;
    }
    st->prev_rms = st->rms;
}

__global__ void k_icp_fix_ns(int *ns, int stride) { *ns = (*ns + stride - 1) / stride; }

__global__ void k_icp_out(const IcpState *s, double *o)
{
    for (int i = 0; i < 12; ++i) o[i] = s->T[i];
    o[12] = s->rms;
    o[13] = s->iters;
    o[14] = s->converged;
    o[15] = s->npairs;
}

// ---------------------------------------------------------------- host side
size_t icp_workspace_bytes(int ns, int nt)
{
    unsigned ht = 1;
    while (ht < 2u * (unsigned)(nt > 0 ? nt : 1)) ht <<= 1;
    const int nbs = (ns + IC_T - 1) / IC_T, nbt = (nt + IC_T - 1) / IC_T;
    size_t b = 0;
    auto add = [&](size_t x) { b += (x + 255) & ~(size_t)255; };
    add(sizeof(double) * 3 * (size_t)(ns > 0 ? ns : 1));  // S
    add(sizeof(double) * 3 * (size_t)(nt > 0 ? nt : 1));  // Q
    add(sizeof(int) * (size_t)(nbs + nbt + 4));           // block counts + totals
    add(sizeof(unsigned long long) * ht);
    add(sizeof(unsigned) * (ht * 3 + 1));
    add(sizeof(double4) * (size_t)(nt > 0 ? nt : 1));
    add(sizeof(int) * (size_t)(ns > 0 ? ns : 1));         // match
    add(sizeof(double) * (size_t)(ns > 0 ? ns : 1));      // dist2
    add(sizeof(double) * 9 * 1024);                       // partials
    add(sizeof(IcpState));
    return b;
}

cudaError_t launch_icp(const float *src, int ns, const float *tgt, int nt, const double init[12], int max_iter,
                       double max_dist, double eps, int stride, void *ws, double *out, cudaStream_t st)
{
    unsigned ht = 1;
    while (ht < 2u * (unsigned)(nt > 0 ? nt : 1)) ht <<= 1;
    const int nbs = (ns + IC_T - 1) / IC_T, nbt = (nt + IC_T - 1) / IC_T;
    char *p = (char *)ws;
    auto take = [&](size_t x) {
        char *r = p;
        p += (x + 255) & ~(size_t)255;
        return r;
    };
    double *S = (double *)take(sizeof(double) * 3 * (size_t)(ns > 0 ? ns : 1));
    double *Q = (double *)take(sizeof(double) * 3 * (size_t)(nt > 0 ? nt : 1));
    int *cnt = (int *)take(sizeof(int) * (size_t)(nbs + nbt + 4));
    int *blks = cnt, *blkt = cnt + nbs, *ns_d = cnt + nbs + nbt, *nt_d = ns_d + 1;
    IcpGrid g;
    g.keys = (unsigned long long *)take(sizeof(unsigned long long) * ht);
    g.count = (unsigned *)take(sizeof(unsigned) * (ht * 3 + 1));
    g.start = g.count + ht;
    g.cursor = g.start + ht;
    g.total = g.cursor + ht;
    g.pts = (double4 *)take(sizeof(double4) * (size_t)(nt > 0 ? nt : 1));
    g.mask = ht - 1;
    g.inv_cell = 1.0 / max_dist;
    g.cell = max_dist;
    int *match = (int *)take(sizeof(int) * (size_t)(ns > 0 ? ns : 1));
    double *dist2 = (double *)take(sizeof(double) * (size_t)(ns > 0 ? ns : 1));
    double *part = (double *)take(sizeof(double) * 9 * 1024);
    IcpState *state = (IcpState *)take(sizeof(IcpState));

    IcpState h;
    memset(&h, 0, sizeof h);
    for (int k = 0; k < 12; ++k) h.T[k] = init[k];
    h.prev_rms = INFINITY;
    h.rms = NAN;
    cudaError_t e;
    if ((e = cudaMemcpyAsync(state, &h, sizeof h, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
    // compaction (source with stride, target all valid)
    k_icp_count<<<nbs, IC_T, 0, st>>>(src, ns, blks);
    k_icp_scan<<<1, 1024, 0, st>>>(blks, nbs, ns_d);
    k_icp_count<<<nbt, IC_T, 0, st>>>(tgt, nt, blkt);
    k_icp_scan<<<1, 1024, 0, st>>>(blkt, nbt, nt_d);
    k_icp_compact<<<nbs, IC_T, 0, st>>>(src, ns, blks, stride, S);
    k_icp_compact<<<nbt, IC_T, 0, st>>>(tgt, nt, blkt, 1, Q);
    // the source count after the stride: ceil(valid / stride), on device
    // (k_icp_pair reads *ns_d; fix it up in place)
    k_icp_fix_ns<<<1, 1, 0, st>>>(ns_d, stride);
    // grid
    if ((e = cudaMemsetAsync(g.keys, 0xff, sizeof(unsigned long long) * ht, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(g.count, 0, sizeof(unsigned) * (ht * 3 + 1), st)) != cudaSuccess) return e;
    k_icp_insert<<<148 * 4, IC_T, 0, st>>>(Q, nt_d, g);
    k_icp_alloc<<<148 * 4, IC_T, 0, st>>>(g);
    k_icp_scatter<<<148 * 4, IC_T, 0, st>>>(Q, nt_d, g);
    note_launch(10);
    const int nb = 148 * 4 < 1024 ? 148 * 4 : 1024;
    const double max_d2 = max_dist * max_dist;
    for (int it = 1; it <= max_iter; ++it) {
        k_icp_pair<<<(unsigned)(((long)ns * IC_G + IC_T - 1) / IC_T), IC_T, 0, st>>>(S, ns_d, g, state, max_d2, match, dist2);
        k_icp_sum1<<<nb, IC_T, 0, st>>>(S, ns_d, Q, state, match, dist2, part);
        k_icp_centroid<<<1, IC_T, 0, st>>>(part, nb, state);
        k_icp_sum2<<<nb, IC_T, 0, st>>>(S, ns_d, Q, state, match, part);
        k_icp_solve<<<1, IC_T, 0, st>>>(part, nb, state, it, eps);
        note_launch(5);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // out: T (12), rms, iters, converged, npairs
    k_icp_out<<<1, 1, 0, st>>>(state, out);
    note_launch();
    return cudaGetLastError();
}

}  // namespace vsbp
