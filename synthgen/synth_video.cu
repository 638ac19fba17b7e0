// synth_video.cu -- device twin of synthgen/video.py (the seeded synthetic UAV
// video of the C5 stream).  INPUT GENERATION ONLY: no arithmetic of the method.
// Bit-identical to the numpy twin (integer arithmetic on lowbias32 hashes); the
// tests compare the two on small frames.  Built into synthgen/libsynth.so, which
// the product library never links.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr uint32_t TAG_TEX = 0x7E1, TAG_IID = 0x11D, TAG_HOLE = 0x401E, TAG_BLD = 0xB1D;

__host__ __device__ __forceinline__ uint32_t hash32(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x;
}
__host__ __device__ __forceinline__ uint32_t mix(uint32_t h, uint32_t v) { return hash32(h ^ v); }

struct Scene {
    uint32_t seed;
    int W, H, s, dmin, dmax, top, W_lo, H_lo, BW;
};

__device__ __forceinline__ int ground(const Scene &c, int y) { return c.dmin + ((c.top - c.dmin) * (y / c.s)) / c.H_lo; }

__device__ int world_label(const Scene &c, long long X, int y)
{
    const long long j = X / c.BW;
    const uint32_t h = mix(hash32(c.seed ^ TAG_BLD), (uint32_t)j);
    const int Wb = c.BW / c.s, Hl = c.H_lo;
    int bw = max(Wb / 6, 1) + (int)(mix(h, 1) % (uint32_t)max(Wb / 3, 1));
    bw = min(bw, Wb);
    int bh = max(Hl / 12, 1) + (int)(mix(h, 2) % (uint32_t)max(Hl / 6, 1));
    bh = min(bh, Hl);
    const int x0 = (int)(mix(h, 3) % (uint32_t)max(Wb - bw + 1, 1));
    const int y0 = (int)(mix(h, 4) % (uint32_t)max(Hl - bh + 1, 1));
    const int height = 4 + (int)(mix(h, 5) % 9u);
    const long long xr = X - j * c.BW;
    const bool inside = xr >= (long long)c.s * x0 && xr < (long long)c.s * (x0 + bw) && y >= c.s * y0 &&
                        y < c.s * (y0 + bh);
    return ground(c, y) + (inside ? height : 0);
}

__global__ void __launch_bounds__(256) k_synth_frames(Scene c, int k0, int n, uint8_t *__restrict__ out)
{
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long per = (long long)c.W * c.H;
    if (idx >= per * n) return;
    const int f = (int)(idx / per);
    const int pix = (int)(idx - (long long)f * per);
    const int y = pix / c.W, x = pix - y * c.W;
    const int k = k0 + f;
    // the world point this pixel sees: largest label whose ray lands on itself
    const int g = ground(c, y);
    int lab = -1;
    long long Xv = 0;
    for (int hgt = 0; hgt <= 12; hgt = hgt == 0 ? 4 : hgt + 1) {
        const int cl = g + hgt;
        const long long X = x + (long long)k * c.s * cl;
        if (world_label(c, X, y) == cl) {
            lab = cl;
            Xv = X;
        }
    }
    uint8_t rgb[3];
    if (lab < 0) {
        const uint32_t hh = mix(mix(mix(hash32(c.seed ^ TAG_HOLE), (uint32_t)k), (uint32_t)x), (uint32_t)y);
        for (int ch = 0; ch < 3; ++ch) rgb[ch] = (uint8_t)(mix(hh, (uint32_t)ch) & 255u);
    } else {
        const int cells[5] = {64, 32, 16, 8, 4}, amps[5] = {16, 8, 4, 2, 1};
        for (int ch = 0; ch < 3; ++ch) {
            const uint32_t hc = mix(hash32(c.seed ^ TAG_TEX), (uint32_t)ch);
            long long total = 0;
#pragma unroll
            for (int o = 0; o < 5; ++o) {
                const int cs = cells[o];
                const uint32_t ho = mix(hc, (uint32_t)o);
                const long long lx = Xv / cs;
                const int fx = (int)(Xv - lx * cs);
                const int ly = y / cs, fy = y - ly * cs;
                const int wx1 = 2 * fx + 1, wy1 = 2 * fy + 1, wx0 = 2 * cs - wx1, wy0 = 2 * cs - wy1;
                const uint32_t hx0 = mix(ho, (uint32_t)lx), hx1 = mix(ho, (uint32_t)(lx + 1));
                const int v00 = (int)(mix(hx0, (uint32_t)ly) & 255u), v10 = (int)(mix(hx1, (uint32_t)ly) & 255u);
                const int v01 = (int)(mix(hx0, (uint32_t)(ly + 1)) & 255u);
                const int v11 = (int)(mix(hx1, (uint32_t)(ly + 1)) & 255u);
                const long long acc = (long long)v00 * wx0 * wy0 + (long long)v10 * wx1 * wy0 +
                                      (long long)v01 * wx0 * wy1 + (long long)v11 * wx1 * wy1;
                total += amps[o] * acc * (4096 / (cs * cs));
            }
            const long long base = (total + 31 * 8192) / (31 * 16384);
            const uint32_t hi = mix(mix(mix(hash32(c.seed ^ TAG_IID), (uint32_t)ch), (uint32_t)Xv), (uint32_t)y);
            const long long v = base + (long long)(hi % 17u) - 8;
            rgb[ch] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
        }
    }
    uint8_t *o = out + idx * 3;
    o[0] = rgb[0];
    o[1] = rgb[1];
    o[2] = rgb[2];
}

}  // namespace

extern "C" {

// frames k0 .. k0+n-1 of the video (seed, W x H, downsample s, labels dmin..dmax)
// into out: u8 [n][H][W][3] device memory; async on `stream`.  0 ok, -1 bad args,
// -4 CUDA error.
int synth_video_frames(uint32_t seed, int W, int H, int s, int dmin, int dmax, int k0, int n, uint8_t *out,
                       void *stream)
{
    if (W < 1 || H < 1 || s < 1 || W % s || H % s || dmin < 0 || dmax < dmin || k0 < 0 || n < 0 || !out) return -1;
    if (n == 0) return 0;
    Scene c;
    c.seed = seed;
    c.W = W;
    c.H = H;
    c.s = s;
    c.dmin = dmin;
    c.dmax = dmax;
    c.top = dmax - 12 > dmin ? dmax - 12 : dmin;
    c.W_lo = W / s;
    c.H_lo = H / s;
    c.BW = s * (c.W_lo / 2 > 1 ? c.W_lo / 2 : 1);
    const long long total = (long long)W * H * n;
    k_synth_frames<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(c, k0, n, out);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // extern "C"
