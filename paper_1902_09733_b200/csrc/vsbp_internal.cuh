// vsbp_internal.cuh -- device-side layout helpers shared by the vsbp kernels.
//
// HBM layout of one pyramid level l (W_l x H_l, Wc = ceil(W_l/2)), DESIGN.md §7:
//   pixels are split by checkerboard colour c = (x+y)&1 (R-10) and stored
//   compactly per row: pixel (x,y) -> (c, y, i = x>>1).  A colour-c iteration
//   then reads only colour 1-c messages and writes only colour c ones, both as
//   contiguous runs along i.
//   cost  D_l : [B][2][H_l][Wc][Lp]       element type TD_l (u8/u16/i32 per level)
//   msgs  M_l : [B][2][4][H_l][Wc][Lp]    element type TM (u8/u16/i32)
//   M_l[b][c][k][y][i][d] = message that pixel (x,y) SENDS toward direction k
//   (0 up, 1 down, 2 left, 3 right).  Lp = L rounded up to 16; labels >= L are 0.
// Each thread owns one 16-label chunk of one pixel: a 16-byte vector at u8,
// 32 bytes at u16, 64 bytes at i32.  The G = pow2 >= Lp/16 threads of one pixel
// are adjacent lanes of a warp.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vsbp {

constexpr int CH = 16;                       // labels per thread chunk
constexpr int BIG = 0x7FF00000;              // > any belief (bp_create bound, R-25)
constexpr unsigned FULL = 0xffffffffu;

__host__ __device__ __forceinline__ size_t d_off(int b, int c, int y, int i, int H, int Wc, int Lp)
{
    return ((((size_t)b * 2 + c) * H + y) * Wc + i) * (size_t)Lp;
}

__host__ __device__ __forceinline__ size_t m_off(int b, int c, int k, int y, int i, int H, int Wc, int Lp)
{
    return (((((size_t)b * 2 + c) * 4 + k) * H + y) * Wc + i) * (size_t)Lp;
}

// ---------------------------------------------------------------- 16-label chunk I/O
// Storage order inside a 16-label chunk (u8 and u16 only; i32 is natural):
//   u8 : byte 4q+b holds label 2q + (b&1) + 8*(b>>1)   (q = 0..3)
//   u16: element 2j+h holds label j + 8h                (j = 0..7)
// so that one PRMT (u8) or nothing (u16) yields the packed u16x2 registers
// r_j = (label j | label j+8 << 16) the fast kernel computes on.  load()/store()
// below convert to/from natural label order v[0..15].
__host__ __device__ __forceinline__ int u8_pos_of_label(int l)
{
    const int r = l & 7;
    return 4 * (r >> 1) + (r & 1) + 2 * (l >> 3);
}
__host__ __device__ __forceinline__ int u16_pos_of_label(int l) { return 2 * (l & 7) + (l >> 3); }

template <typename T> struct Chunk;

template <> struct Chunk<uint8_t> {
    static __device__ __forceinline__ void load(const uint8_t *p, int v[CH])
    {
        uint4 w = __ldg(reinterpret_cast<const uint4 *>(p));
        unsigned u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            v[2 * q] = u[q] & 0xff;
            v[2 * q + 1] = (u[q] >> 8) & 0xff;
            v[2 * q + 8] = (u[q] >> 16) & 0xff;
            v[2 * q + 9] = u[q] >> 24;
        }
    }
    static __device__ __forceinline__ void store(uint8_t *p, const int v[CH])
    {
        unsigned u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            u[q] = (unsigned)v[2 * q] | ((unsigned)v[2 * q + 1] << 8) | ((unsigned)v[2 * q + 8] << 16) |
                   ((unsigned)v[2 * q + 9] << 24);
        *reinterpret_cast<uint4 *>(p) = make_uint4(u[0], u[1], u[2], u[3]);
    }
};

template <> struct Chunk<uint16_t> {
    static __device__ __forceinline__ void load(const uint16_t *p, int v[CH])
    {
        const uint4 *q4 = reinterpret_cast<const uint4 *>(p);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint4 w = __ldg(q4 + h);
            unsigned u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                v[4 * h + q] = u[q] & 0xffff;
                v[4 * h + q + 8] = u[q] >> 16;
            }
        }
    }
    static __device__ __forceinline__ void store(uint16_t *p, const int v[CH])
    {
        uint4 *q4 = reinterpret_cast<uint4 *>(p);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            unsigned u[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) u[q] = (unsigned)v[4 * h + q] | ((unsigned)v[4 * h + q + 8] << 16);
            q4[h] = make_uint4(u[0], u[1], u[2], u[3]);
        }
    }
};

template <> struct Chunk<int32_t> {
    static __device__ __forceinline__ void load(const int32_t *p, int v[CH])
    {
        const int4 *q4 = reinterpret_cast<const int4 *>(p);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            int4 w = __ldg(q4 + h);
            v[4 * h] = w.x;
            v[4 * h + 1] = w.y;
            v[4 * h + 2] = w.z;
            v[4 * h + 3] = w.w;
        }
    }
    static __device__ __forceinline__ void store(int32_t *p, const int v[CH])
    {
        int4 *q4 = reinterpret_cast<int4 *>(p);
#pragma unroll
        for (int h = 0; h < 4; ++h) q4[h] = make_int4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
    }
};

// storage index of label d (any chunk) for element type T
template <typename T> __device__ __forceinline__ int pos_of_label(int d)
{
    if (sizeof(T) == 1) return (d & ~15) + u8_pos_of_label(d & 15);
    if (sizeof(T) == 2) return (d & ~15) + u16_pos_of_label(d & 15);
    return d;
}

__device__ __forceinline__ void zero16(int v[CH])
{
#pragma unroll
    for (int j = 0; j < CH; ++j) v[j] = 0;
}

// thread-local launch accounting (host side)
void note_launch(int n = 1);

}  // namespace vsbp
