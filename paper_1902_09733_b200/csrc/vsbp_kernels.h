// vsbp_kernels.h -- host-side launchers of the vsbp kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vsbp {

// Geometry of one launch: the level being processed (W,H,Wc) and, where used,
// its parent level (Wp,Hp,Wcp); label padding and the lane-group width G.
struct Geom {
    int B;
    int W, H, Wc;
    int Wp, Hp, Wcp;
    int L, Lp, nch, G, log2G;
};

cudaError_t launch_costvol(const uint8_t *left, const uint8_t *right, void *D, int dbytes, const Geom &g, int lam_q,
                           int tau_d, cudaStream_t st);
// fused cost volume + pyramid levels 0..F-1 (costpyr.cu), F <= 5
struct CostPyrArgs {
    void *D[5];
    int dbytes[5];
    int W[5], H[5], Wc[5];
    size_t pairD[5];  // elements per pair of level l's cost array
    int L, Lp, nch, F;
    int lam_q, tau_d;
    int write0;       // write level 0 (0: only the coarser levels are stored)
    int img_smem;     // set by the launcher
};
size_t costpyr_smem(int L, int Lp, int F);
cudaError_t launch_costpyr(const uint8_t *left, const uint8_t *right, CostPyrArgs a, int B, cudaStream_t st);
cudaError_t launch_pyramid(const void *Dc, int cbytes, void *Dp, int pbytes, const Geom &g, cudaStream_t st);
cudaError_t launch_update(const void *D, int dbytes, void *M, const void *Mp, int mbytes, const Geom &g, int mode,
                          int colour, int S, int tau_q, cudaStream_t st);
cudaError_t launch_upcopy(void *M, const void *Mp, int mbytes, const Geom &g, int colour, cudaStream_t st);
cudaError_t launch_wta(const void *D, int dbytes, const void *M, int mbytes, const Geom &g, int32_t *disp,
                       int only_colour, cudaStream_t st);
// arguments of the packed update kernel (bp_fast.cu); offsets are per pair, in elements
struct FastArgs {
    uint8_t *M;        // this level's messages
    uint8_t *Mw;       // k_update_pair: the level's other message array (colour-B output)
    const uint8_t *Mp; // parent level's messages (MODE 2)
    int32_t *disp;     // WTA output (fused WTA / MODE 3)
    uint32_t npix;     // H * Wc (pixels of one colour)
    uint32_t magic;    // ceil(2^32 / Wc) when exact for every pixel index, else 0
    int W, H, Wc, Wp, Hp, Wcp;
    int L, Lp, nch, G, log2G;
    uint32_t colour;
    uint32_t plane, planep;  // H*Wc*Lp, Hp*Wcp*Lp
    size_t pairD, pairM, pairMp;
    uint32_t SS, TT;         // S and tau_q replicated in both 16-bit halves
    // level 0 with dbytes == 0: the data term is computed from the grey images
    const uint8_t *gl, *gr;  // [B][H][W]
    size_t img_elems;        // B*H*W (bounds of the vector loads)
    uint32_t lam, T2d;       // lambda_q; tau_d in both 16-bit halves
};
// dbytes 1 / 2: D is u8 / u16; dbytes 0: level 0 computed from a.gl / a.gr (ImgD)
cudaError_t launch_update_fast(const void *D, int dbytes, const FastArgs &a, int B, int mode, bool wta, bool sgn,
                               cudaStream_t st);
// two checkerboard iterations (a.colour, then its complement) in one launch, reading
// a.M (or the parent, mode 2; nothing, mode 1) and writing the second colour's
// messages to a.Mw; rows per CTA band
cudaError_t launch_update_pair(const void *D, int dbytes, const FastArgs &a, int B, int mode, bool sgn, int band,
                               cudaStream_t st, bool fin = false);
size_t pair_smem_bytes(int dbytes);
// fused last level-0 iteration + WTA of both colours (a.colour = the colour updated last)
cudaError_t launch_final_fast(const void *D, const FastArgs &a, int B, bool sgn, cudaStream_t st);
cudaError_t launch_final_tile(const void *D, const FastArgs &a, int B, bool sgn, cudaStream_t st);
cudaError_t launch_export_msgs(const void *M, int mbytes, const Geom &g, int b, int32_t *out, cudaStream_t st);
cudaError_t launch_export_costs(const void *D, int dbytes, const Geom &g, int b, int32_t *out, cudaStream_t st);

// tile_cnt (optional): also count the pixels with D >= min_disp per a8 compaction
// segment (128 pixels of a row, compact.cu; zeroed first), for launch_compact_from_counts
cudaError_t launch_jbu_fast(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide, int s, float *disp_hi,
                            float sigma_s, float sigma_r, int radius, const float *Qf, float min_disp, float *xyz,
                            unsigned long long *n_valid, cudaStream_t st, int *tile_cnt = nullptr);
cudaError_t launch_reproject(int B, const float *disp, int W, int H, const float Qf[16], float min_disp, float *xyz,
                             unsigned long long *n_valid, cudaStream_t st);
cudaError_t launch_prep(int n, const uint8_t *rgb, int W_hi, int H_hi, int s, uint8_t *gray, cudaStream_t st);
// a8 compaction (compact.cu)
size_t compact_workspace_bytes(int B, int W, int H);
int compact_tiles_per_pair(int W, int H);  // segments (128-pixel row pieces) per pair
int compact_segs_per_row(int W);
int *compact_counts(void *ws);
cudaError_t compact_zero_counts(int B, int W, int H, void *ws, cudaStream_t st);
cudaError_t launch_compact_from_counts(int B, const float *disp, int W, int H, const float Qf[16], float min_disp,
                                       float *xyz, long long cap, long long *offsets, unsigned long long *n_valid,
                                       void *ws, cudaStream_t st);
cudaError_t launch_compact(int B, const float *disp, int W, int H, const float Qf[16], float min_disp, float *xyz,
                           long long cap, long long *offsets, unsigned long long *n_valid, void *ws,
                           cudaStream_t st);
cudaError_t launch_summary(int B, const int32_t *disp, int W, int H, const unsigned long long *n_valid,
                           uint64_t first_pair_id, void *summary, cudaStream_t st);

}  // namespace vsbp

namespace vsbp {
// row f1 (rectify.cu): radial undistortion + bilinear remap fused with a0
bool rectify_domain_ok(int W, int H, const double *cam);
cudaError_t launch_rectify_prep(int n, const uint8_t *raw, int W, int H, const double *cam, int s, uint8_t *gray,
                                uint8_t *rect, cudaStream_t st);
}  // namespace vsbp

namespace vsbp {
// row f3 (features.cu): Harris response + grid selection, ZSSD matching
cudaError_t launch_harris(int n, const uint8_t *img, int W, int H, int gc, int gr, int K, int64_t thr, int64_t *R25,
                          int32_t *xy, int64_t *resp, int32_t *count, cudaStream_t st);
size_t zssd_smem(int r, int sr);
cudaError_t launch_zssd_match(int n, const uint8_t *img1, const uint8_t *img2, int W, int H, const int32_t *xy,
                              int ncorner, int r, int sr, int64_t max_cost, int32_t *match, int64_t *mcost,
                              cudaStream_t st);
}  // namespace vsbp

namespace vsbp {
// row f2 (csbp.cu): constant-space BP
constexpr int CS_KMAX = 64;  // candidates per pixel handled by the kernels
struct CsbpArgs {
    int W, H, L;             // level-0 (full BP resolution) image and labels
    int lam_q, tau_d, tau_q, S;
};
struct CsbpLevel {
    int l, W, H, n, k;       // level index, dims, pixels, candidates per pixel
    uint16_t *cand;          // [B][n][k] ascending labels
    int32_t *dsel;           // [B][n][k] data cost of each candidate at this level
    int32_t *msg;            // [B][n][4][k] incoming (receiver-stored) messages
};
cudaError_t launch_csbp_top(const uint8_t *left, const uint8_t *right, const CsbpArgs &a, const CsbpLevel &lv, int B,
                            cudaStream_t st);
cudaError_t launch_csbp_init(const uint8_t *left, const uint8_t *right, const CsbpArgs &a, const CsbpLevel &lv,
                             const CsbpLevel &pv, int B, cudaStream_t st);
cudaError_t launch_csbp_update(const CsbpArgs &a, const CsbpLevel &lv, int colour, int B, cudaStream_t st);
cudaError_t launch_csbp_wta(const CsbpLevel &lv, int32_t *disp, int B, cudaStream_t st);
cudaError_t launch_csbp_export(const uint16_t *cand, size_t n, int32_t *out, cudaStream_t st);
}  // namespace vsbp

namespace vsbp {
// row f4 (icp.cu): point-to-point ICP in float64
size_t icp_workspace_bytes(int ns, int nt);
cudaError_t launch_icp(const float *src, int ns, const float *tgt, int nt, const double init[12], int max_iter,
                       double max_dist, double eps, int stride, void *ws, double *out, cudaStream_t st);
}  // namespace vsbp
