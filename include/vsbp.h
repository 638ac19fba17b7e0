/*
 * vsbp.h -- C ABI of the B200-native stereo hot path of arXiv 1902.09733
 *           ("Towards Real-time 3D Reconstruction using Consumer UAVs").
 *
 * Library: paper_1902_09733_b200/libvsbp.so (sm_100a CUDA kernels + host glue).
 * Citations: P:n = PAPER.md line n; R-n = reading n in DESIGN.md §3.
 *
 * Conventions for every entry point
 *   - Buffer pointers are DEVICE pointers unless stated otherwise, owned by the
 *     caller, row-major and tightly packed.  The library never allocates device
 *     memory: scratch space is a caller-provided workspace (bp_set_workspace).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Every call only ENQUEUES work on that stream and never synchronises the
 *     host; results are ready when the stream reaches that point.
 *   - Return value: 0 on success, a negative VSBP_E* code on failure.  The
 *     library never throws, aborts or prints; vsbp_strerror() describes a code
 *     (for VSBP_ECUDA it carries the last CUDA error string of the calling thread).
 *   - A context (vsbp_bp) may be used by one stream at a time; distinct contexts
 *     are independent.
 *   - There is no CPU implementation behind this ABI: without a B200 every
 *     compute call returns VSBP_ECUDA.
 */
#ifndef VSBP_H
#define VSBP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VSBP_OK 0
#define VSBP_EINVAL (-1)    /* null pointer, out-of-range size or parameter */
#define VSBP_EDIM (-2)      /* dimension mismatch, workspace too small, batch > planned */
#define VSBP_EOVERFLOW (-3) /* int32 fixed-point bound violated (see bp_create) */
#define VSBP_ECUDA (-4)     /* CUDA launch/driver error (see vsbp_strerror) */

typedef struct vsbp_bp vsbp_bp; /* opaque BP context */

/* Per-pair summary written by pair_summary (a8): 64 bytes, device memory. */
typedef struct vsbp_summary {
    uint64_t n_valid;    /* points with d >= min_disp (reproject)              */
    int64_t label_sum;   /* sum of low-res disparity labels                    */
    uint64_t label_hash; /* sum_i mix64(i<<32 | label_i) mod 2^64  */
    uint64_t pair_id;    /* caller's pair index                                */
    uint64_t reserved[4];
} vsbp_summary;

/* ---------------------------------------------------------------------------
 * bp_create -- plan hierarchical min-sum BP (§2.2 Eq.1, §3.2).
 *   W, H      : BP resolution (the downsampled pair), W,H >= 1
 *   ndisp     : number of labels L, disparities d in [0, L), 2 <= L <= 512
 *   levels    : pyramid levels (1 = flat BP), 1 <= levels <= 16 (R-12)
 *   iters     : checkerboard iterations per level (one iteration = one colour,
 *               R-10), >= 1
 *   lambda    : data-term weight (R-5), >= 0
 *   data_trunc: truncation of |L - R| in intensity levels (R-2), rounds to >= 1
 *   disc_trunc: smoothness truncation in labels (R-3), rounds to >= 1/128
 * Fixed point (R-6): S = 128, lambda_q = rha(lambda*S), tau_d = rha(data_trunc),
 * tau_q = rha(disc_trunc*S).
 * Errors: VSBP_EINVAL for out-of-range arguments; VSBP_EOVERFLOW when
 *   lambda_q*tau_d*4^(levels-1) + 4*tau_q + 2^20 >= 2^31 (R-25).
 * Host-only; allocates only host metadata.  *out receives the context.
 * ------------------------------------------------------------------------- */
int bp_create(int W, int H, int ndisp, int levels, int iters, float lambda, float data_trunc,
              float disc_trunc, vsbp_bp **out);

/* Options (measurement / parity knobs); call before bp_set_workspace.
 *   VSBP_OPT_MSG_BYTES : message storage width in bytes, 0 = narrowest lossless
 *                        (u8 if tau_q <= 255, u16 if <= 65535, else 4), 1, 2 or 4;
 *                        narrower than lossless -> VSBP_EINVAL.
 *   VSBP_OPT_KERNEL    : 0 = fastest available kernels (packed message update,
 *                        fused cost volume + pyramid), 1 = generic kernels
 *                        (same results, bit for bit). */
#define VSBP_OPT_MSG_BYTES 1
#define VSBP_OPT_KERNEL 2
/*   VSBP_OPT_DIMG      : 1 = the packed kernel computes the level-0 data term from
 *                        the grey images inside the message update, so D_0 is
 *                        neither stored nor read (bp_get_costs rebuilds it on demand
 *                        from the last call's images); 0 (default) = store and read
 *                        D_0.  2 = only the one-iteration level-0 launches compute it
 *                        (D_0 still stored for the two-iteration kernel).  Results
 *                        are identical; both trade level-0 bytes for ALU work and
 *                        measured slower. */
#define VSBP_OPT_DIMG 3
/*   VSBP_OPT_FINAL     : 1, 2 or 3 = the last level-0 iteration is fused with the WTA
 *                        of both colours: its messages go straight into the
 *                        receivers' beliefs and are never stored, so
 *                        bp_get_messages(level 0) returns VSBP_EINVAL after such a
 *                        call.  1: each colour-B pixel recomputes its neighbours'
 *                        messages (k_final_fast); 2: tiles keep the messages in
 *                        shared memory (k_final_tile); 3: the two-iteration
 *                        kernel's row wavefront -- the A-phase updates and labels
 *                        colour A, the B-phase labels colour B from the on-chip
 *                        messages (the pipeline's setting).  0 (default) = store
 *                        them and label in separate passes.  Disparities are
 *                        identical; 1 and 2 measured slower.
 *                        Applies when the packed kernels run with u8 level-0
 *                        costs, iters >= 2 and W >= 2 (3: also L <= 32 * 16,
 *                        i.e. lane groups of at most 32). */
#define VSBP_OPT_FINAL 4
/*   VSBP_OPT_PAIR      : 1 (default) = two checkerboard iterations per launch on
 *                        large levels where the packed kernel runs with
 *                        D from memory and the level has >= 3 iterations (all but
 *                        its last iteration go in pairs): the first colour's
 *                        messages stay on chip, so a pair moves 10L instead of 18L
 *                        bytes per pixel pair at u8 (levels with u8 costs and >=
 *                        VSBP_OPT_PAIR_MINPX pixels; levels with u16 costs and
 *                        >= 10000 pixels when the call's batch holds >= 2M of
 *                        their pixels).  The level's messages then alternate
 *                        between two arrays (bp_workspace_bytes grows by one
 *                        message array per such level at the workspace's batch).
 *                        2 = on every eligible level (tests); 3 = u8-cost levels
 *                        only; 0 = one iteration per launch.  Results are
 *                        identical.
 *   VSBP_OPT_PAIR_BAND : rows per CTA of the two-iteration kernel (default 64;
 *                        levels shorter than two bands use 16).
 *   VSBP_OPT_PAIR_MINPX: smallest level (W_l * H_l pixels) fused under
 *                        VSBP_OPT_PAIR = 1 (default 100000). */
#define VSBP_OPT_PAIR 5
#define VSBP_OPT_PAIR_BAND 6
#define VSBP_OPT_PAIR_MINPX 7
int bp_set_option(vsbp_bp *ctx, int option, int value);

/* Quantised parameters: out[0..7] = {lambda_q, tau_d, tau_q, S, msg_bytes,
 * labels padded (Lp), levels, iters}. */
int bp_get_params(const vsbp_bp *ctx, int32_t out[8]);

/* Dimensions of pyramid level `level` (ceil-halving, R-12). */
int bp_level_dims(const vsbp_bp *ctx, int level, int *W, int *H);

/* Device scratch needed for `batch` pairs, and binding it (caller-owned,
 * 256-byte aligned, must outlive every call that uses it). */
size_t bp_workspace_bytes(const vsbp_bp *ctx, int batch);
int bp_set_workspace(vsbp_bp *ctx, void *dptr, size_t bytes, int batch);

/* ---------------------------------------------------------------------------
 * bp_disparity_batch -- a1..a5 for B independent pairs.
 *   left, right : u8 [B][H][W] rectified, downsampled grey pairs
 *   disp        : int32 [B][H][W] labels, the WTA argmin of Eq.1's E_X(d)
 *                 (P:34), ties -> smallest d (R-13)
 * Requires a workspace bound for >= B pairs (else VSBP_EDIM).
 * The per-level message fields stay in the workspace for bp_get_messages
 * (level 0 only with VSBP_OPT_FINAL = 0).
 * bp_disparity is the B = 1 case.
 * ------------------------------------------------------------------------- */
int bp_disparity_batch(vsbp_bp *ctx, int B, const uint8_t *left, const uint8_t *right, int32_t *disp,
                       void *stream);
int bp_disparity(vsbp_bp *ctx, const uint8_t *left, const uint8_t *right, int32_t *disp, void *stream);

/* Debug / parity export after bp_disparity*: the final messages of `level` for
 * pair `pair`, as int32 [4][H_l][W_l][L] with M[k][y][x][d] = message pixel
 * (x,y) sends toward direction k (0 up, 1 down, 2 left, 3 right); and the cost
 * pyramid level as int32 [H_l][W_l][L]. */
int bp_get_messages(vsbp_bp *ctx, int pair, int level, int32_t *out, void *stream);
int bp_get_costs(vsbp_bp *ctx, int pair, int level, int32_t *out, void *stream);

void bp_destroy(vsbp_bp *ctx);

/* ---------------------------------------------------------------------------
 * jbu_upsample_batch -- a6, joint bilateral upsampling (Eq.2; R-15..R-19,
 * R-24).  For B pairs:
 *   disp_lo   : int32 [B][H][W] low-res labels
 *   guide_rgb : u8 [B][s*H][s*W][3] full-res colour guide (the left frame, R-17)
 *   disp_hi   : float [B][s*H][s*W] upsampled disparity in FULL-RES pixels (x s)
 *   sigma_s   : spatial sigma in LOW-RES pixels, with
 *               log2(e)*(radius+0.5)^2/sigma_s^2 <= 100 (else VSBP_EINVAL: the
 *               window's weights would leave f32 range); sigma_r: range sigma on
 *               the 0..255 scale (> 0); radius: window half-width in low-res
 *               pixels, 1..8; s: integer scale 1..16.
 * Accuracy: agrees with the double oracle within 1e-4 full-res px for every
 * output below 2048 px, and within one f32 ulp of it above (the float output
 * cannot be closer there), for any int32 labels |D'| < 2^24.  Windows whose
 * label spread times s is at most 256 run in f32 on residual labels
 * (D'_q - D'_centre; error ~2e-7 * s * spread); wider windows are computed with
 * double weights and sums (slower, rare on smooth maps).
 * jbu_upsample is the B = 1 case.
 * ------------------------------------------------------------------------- */
int jbu_upsample_batch(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide_rgb, int s,
                       float *disp_hi, float sigma_s, float sigma_r, int radius, void *stream);
int jbu_upsample(const int32_t *disp_lo, int W, int H, const uint8_t *guide_rgb, int s, float *disp_hi,
                 float sigma_s, float sigma_r, int radius, void *stream);

/* ---------------------------------------------------------------------------
 * jbu_reproject_batch -- a6 + a7 fused (the pipeline's call): jbu_upsample_batch
 * followed by reproject_batch on its output, in one kernel, without re-reading
 * disp_hi.  Arguments as in those two calls; xyz : float [B][s*H][s*W][3];
 * n_valid : device uint64 [B], overwritten.  Errors: the union of both calls'.
 * ------------------------------------------------------------------------- */
int jbu_reproject_batch(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide_rgb, int s,
                        float sigma_s, float sigma_r, int radius, const double *Q, float min_disp,
                        float *disp_hi, float *xyz, unsigned long long *n_valid, void *stream);

/* ---------------------------------------------------------------------------
 * reproject_batch -- a7, Eq.3 (R-20, R-21):
 *   [X Y Z Wh]^T = Q [u v d 1]^T, xyz = (X,Y,Z)/Wh if d >= min_disp else NaN.
 *   disp    : float [B][H][W] full-res disparity (px)
 *   Q       : HOST pointer, double[16] row-major (copied at call time)
 *   xyz     : float [B][H][W][3]
 *   n_valid : device uint64 [B]; overwritten with the count of valid points.
 * min_disp <= 0 -> VSBP_EINVAL.  reproject is the B = 1 case.
 * ------------------------------------------------------------------------- */
int reproject_batch(int B, const float *disp, int W, int H, const double *Q, float min_disp, float *xyz,
                    unsigned long long *n_valid, void *stream);
int reproject(const float *disp, int W, int H, const double *Q, float min_disp, float *xyz,
              unsigned long long *n_valid, void *stream);

/* ---------------------------------------------------------------------------
 * vsbp_q_matrix -- Eq.3 as the 4x4 matrix reproject* take, with the
 * printed z = (B/d)(f B/du) read as z = f_du B / d (R-20, the only form that
 * inverts Eq.3's first line):
 *   Q = [[1, 0, 0, -u0], [0, f_du/f_dv, 0, -v0 f_du/f_dv], [0, 0, 0, f_du],
 *        [0, 0, 1/B, 0]]   (row-major, written to the HOST double[16] Q)
 * so that x = B(u-u0)/d, y = B(v-v0)(f_du/f_dv)/d, z = f_du B/d.  f_du, f_dv, B
 * must be finite and nonzero (else VSBP_EINVAL).  Host-only.
 * ------------------------------------------------------------------------- */
int vsbp_q_matrix(double f_du, double f_dv, double u0, double v0, double B, double *Q);

/* ---------------------------------------------------------------------------
 * compact_cloud_batch -- a8, the per-pair point cloud as PACKED valid points in
 * raster order (Eq.3 turns each pair's disparity into "a point cloud";
 * SURVEY 8(a) a8; R-20, R-21):
 *   disp      : float [B][H][W] full-res disparity (px), device
 *   Q         : HOST double[16] (as reproject_batch); min_disp > 0
 *   xyz       : float [cap_points][3] device output: the points with
 *               d >= min_disp, pair-major then row-major then column-major, each
 *               bit-identical to reproject's / jbu_reproject_batch's entry
 *   offsets   : device int64 [B+1]: offsets[b] = index of pair b's first point,
 *               offsets[B] = total points (always exact, even past cap_points)
 *   n_valid   : device uint64 [B], overwritten with each pair's count
 *   workspace : device scratch of compact_workspace_bytes(B, W, H) bytes
 * Points at index >= cap_points are not written (cap_points = B*W*H can never
 * overflow).  Count, scan and write kernels; async.
 * Errors: VSBP_EINVAL (null pointers, B < 1, W*H > 2^30, min_disp <= 0, workspace
 * too small or not 256-byte aligned, cap_points < 0).
 * ------------------------------------------------------------------------- */
size_t compact_workspace_bytes(int B, int W, int H);
int compact_cloud_batch(int B, const float *disp, int W, int H, const double *Q, float min_disp, float *xyz,
                        long long cap_points, long long *offsets, unsigned long long *n_valid, void *workspace,
                        size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * jbu_compact_batch -- a6 + a7 + a8, the pipeline's call: jbu_upsample_batch
 * (disp_hi) followed by compact_cloud_batch on its output, with the compaction's
 * count pass folded into the JBU kernel (each valid pixel counted as it is
 * produced) so disp_hi is read back only once.  Arguments as in those two calls;
 * workspace of compact_workspace_bytes(B, s*W, s*H) bytes.  Results identical
 * to the two calls made separately.
 * ------------------------------------------------------------------------- */
int jbu_compact_batch(int B, const int32_t *disp_lo, int W, int H, const uint8_t *guide_rgb, int s, float sigma_s,
                      float sigma_r, int radius, const double *Q, float min_disp, float *disp_hi, float *xyz,
                      long long cap_points, long long *offsets, unsigned long long *n_valid, void *workspace,
                      size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * prep_downsample_batch -- a0 (R-22): for n frames,
 *   rgb_hi : u8 [n][H_hi][W_hi][3]  ->  gray_lo : u8 [n][H_hi/s][W_hi/s]
 *   grey = (77R+150G+29B+128)>>8, then s x s mean rounded half up.
 * W_hi, H_hi must be multiples of s (else VSBP_EDIM).
 * ------------------------------------------------------------------------- */
int prep_downsample_batch(int n, const uint8_t *rgb_hi, int W_hi, int H_hi, int s, uint8_t *gray_lo,
                          void *stream);
int prep_downsample(const uint8_t *rgb_hi, int W_hi, int H_hi, int s, uint8_t *gray_lo, void *stream);

/* ---------------------------------------------------------------------------
 * rectify_prep_batch -- row f1 fused with a0 (§2.1: radial-only
 * undistortion, "cvInitUndistortMap() and cvRemap()"; R-26, R-27):
 *   rgb_raw  : u8 [n][H_hi][W_hi][3] distorted frames (device)
 *   cam      : HOST pointer, double[7] = {f_u, f_v, c_u, c_v, k1, k2, k3} (pixels;
 *              new camera matrix = old, no tangential terms); copied at call time
 *   gray_lo  : u8 [n][H_hi/s][W_hi/s]: grey + s x s box mean (as prep_downsample)
 *              of the undistorted frame
 *   rgb_rect : u8 [n][H_hi][W_hi][3] undistorted frames, or NULL (not written)
 * Destination pixel (u,v) samples the source at the radial map of R-26 quantised
 * to 1/32 px; channels are interpolated with integer bilinear weights (R-27),
 * taps outside the frame read 0.  s in 1..8; W_hi, H_hi multiples of s (else
 * VSBP_EDIM); f_u, f_v <= 0 -> VSBP_EINVAL; a map that can leave |coordinate| <
 * 2^24 px (R-26 bound) -> VSBP_EOVERFLOW.
 * ------------------------------------------------------------------------- */
int rectify_prep_batch(int n, const uint8_t *rgb_raw, int W_hi, int H_hi, const double *cam, int s,
                       uint8_t *gray_lo, uint8_t *rgb_rect, void *stream);

/* ---------------------------------------------------------------------------
 * Constant-space BP -- row f2, the BP the paper cites as [4] ("GPU based
 * Belief Propagation [4]"; [4] = Yang, Wang, Ahuja, CVPR 2010; R-32..R-35).
 * Same energy, quantisation, pyramid and checkerboard schedule as bp_create's BP,
 * but level l keeps only k_l = min(ndisp, k0 * 2^l) candidate labels per pixel:
 * the workspace is O(k) per pixel instead of O(ndisp) and the data term of a
 * candidate is computed from the images on demand.
 *   csbp_create     : arguments as bp_create plus k0 >= 1; VSBP_EINVAL if any
 *                     k_l > 64; VSBP_EOVERFLOW as bp_create.  Host-only.
 *   csbp_workspace_bytes / csbp_set_workspace : as the bp_ equivalents (caller-
 *                     owned device memory, 256-byte aligned).
 *   csbp_disparity_batch : left, right u8 [B][H][W] -> disp int32 [B][H][W] labels;
 *                     async on `stream`.
 *   csbp_get_candidates : debug/parity, level l's candidate labels of one pair as
 *                     int32 [H_l][W_l][k_l] (ascending per pixel).
 * ------------------------------------------------------------------------- */
typedef struct vsbp_csbp vsbp_csbp;
int csbp_create(int W, int H, int ndisp, int levels, int iters, int k0, float lambda, float data_trunc,
                float disc_trunc, vsbp_csbp **out);
size_t csbp_workspace_bytes(const vsbp_csbp *ctx, int batch);
int csbp_set_workspace(vsbp_csbp *ctx, void *dptr, size_t bytes, int batch);
int csbp_disparity_batch(vsbp_csbp *ctx, int B, const uint8_t *left, const uint8_t *right, int32_t *disp,
                         void *stream);
int csbp_get_candidates(vsbp_csbp *ctx, int pair, int level, int32_t *out, void *stream);
void csbp_destroy(vsbp_csbp *ctx);

/* ---------------------------------------------------------------------------
 * icp_register -- row f4, point-to-point ICP between two clouds ("CUDA
 * accelerated Iterative Closest Point (ICP) [6] ... point clouds calculated from
 * low-resolution disparity maps using Equation 3"; R-36):
 *   src, tgt : float [n][3] device clouds (rows with a NaN are ignored, R-21)
 *   init     : HOST double[12], the initial [R|t] (row-major 3x4), e.g. the EPnP
 *              relative pose; max_iter >= 1, max_dist > 0 (m, pairing radius and
 *              grid cell), eps > 0 (rms-change stop), stride >= 1 (source subsample)
 *   ws       : device workspace of icp_workspace_bytes(ns, nt) bytes (256-aligned)
 *   out      : DEVICE double[16] = {R|t (12), rms, iterations (-1: no pairs),
 *              converged (0/1), pairs of the last iteration}
 * Pairing, reductions and the rigid solve run on the device in float64; the
 * max_iter iterations are enqueued without host synchronisation.
 * ------------------------------------------------------------------------- */
size_t icp_workspace_bytes(int ns, int nt);
int icp_register(const float *src, int ns, const float *tgt, int nt, const double *init, int max_iter,
                 double max_dist, double eps, int stride, void *ws, size_t ws_bytes, double *out, void *stream);

/* ---------------------------------------------------------------------------
 * harris_corners_batch -- row f3, Harris corners on a grid (§2.3 Eq.4-5;
 * P:84 "a 30x30 grid ... Harris corners inside each grid individually"; SPEC
 * S:310-316; R-28, R-29), for n grey images:
 *   gray : u8 [n][H][W];  R25 : int64 [n][H][W] workspace/output: 25 * Harris
 *          response (k = 0.04), INT64_MIN outside 3 <= x <= W-4, 3 <= y <= H-4
 *   corners: the K strict 3x3 maxima with 25R >= thr and the largest response in
 *          each of the gc x gr cells (ties to raster order):
 *          xy : int32 [n][gr*gc*K][2], resp : int64 [n][gr*gc*K] (unused slots
 *          {-1,-1} / INT64_MIN), count : int32 [n][gr*gc]
 * W, H >= 9; 1 <= K <= 16; gc, gr >= 1; thr >= 1 (else VSBP_EINVAL).
 * ------------------------------------------------------------------------- */
int harris_corners_batch(int n, const uint8_t *gray, int W, int H, int gc, int gr, int K, long long thr,
                         long long *R25, int32_t *xy, long long *resp, int32_t *count, void *stream);

/* ---------------------------------------------------------------------------
 * zssd_match_batch -- row f3, ZSSD correspondence between two frames ("compute
 * correspondence between frame I_t1 and I_t2 ... within the given search range ...
 * ZSSD"; R-30, R-31), for n image pairs:
 *   img1, img2 : u8 [n][H][W];  xy : int32 [n][ncorner][2] corners of img1 (slots
 *   with x < 0 are skipped);  r : patch radius (1..7);  sr : search radius (1..64)
 *   match : int32 [n][ncorner][2] matched position in img2 or {-1,-1};
 *   cost  : int64 [n][ncorner] n*ZSSD of the match (n = (2r+1)^2) or -1.
 * A match is the least cost over the (2sr+1)^2 window (patch inside img2), ties to
 * raster order, kept iff cost <= max_cost and the least cost beyond Chebyshev
 * distance 2 exceeds 1.2x it (5*second > 6*best) or does not exist.
 * ------------------------------------------------------------------------- */
int zssd_match_batch(int n, const uint8_t *img1, const uint8_t *img2, int W, int H, const int32_t *xy,
                     int ncorner, int r, int sr, long long max_cost, int32_t *match, long long *cost, void *stream);

/* ---------------------------------------------------------------------------
 * pair_summary_batch -- a8: for B pairs write summary[b] =
 *   {n_valid[b], sum of disp_lo[b], label hash of disp_lo[b], first_pair_id + b}.
 *   disp_lo : int32 [B][H][W]; n_valid : device uint64 [B]; summary : device [B].
 * ------------------------------------------------------------------------- */
int pair_summary_batch(int B, const int32_t *disp_lo, int W, int H, const unsigned long long *n_valid,
                       uint64_t first_pair_id, vsbp_summary *summary, void *stream);

/* Live timing of the message-update kernels (a4), for bench.py's roofline.
 * bp_timing_enable(ctx, 1) makes every later bp_disparity* record CUDA events
 * (on the call's stream) around each level's run of update launches;
 * bp_timing_read synchronises those events and returns, accumulated since the
 * last read, per level l < 16: ms[l] = device milliseconds of the level's update
 * launches, launches[l] = number of launches, bytes[l] = their ALGORITHMIC bytes
 * (updated pixels x (L*w_D + 8*L*w_M)).  Host pointers, >= 16 entries. */
int bp_timing_enable(vsbp_bp *ctx, int enable);
int bp_timing_read(vsbp_bp *ctx, double *ms, int64_t *launches, double *bytes);

/* Live timing of the JBU kernel (a6, with the a8 counts) inside jbu_compact_batch,
 * for bench.py's second roofline: jbu_timing_enable(1) makes every later
 * jbu_compact_batch record CUDA events around that kernel on its stream (process-wide;
 * not thread-safe); jbu_timing_read synchronises them and returns, accumulated since
 * the last read, the device ms, the launches and the algorithmic pixel-taps (B * sW *
 * sH * (2r+1)^2: one weight, one 2^x, each).  Errors: VSBP_EINVAL (null pointers),
 * VSBP_ECUDA. */
int jbu_timing_enable(int enable);
int jbu_timing_read(double *ms, long long *launches, double *taps);

const char *vsbp_strerror(int code);

/* Number of kernel launches this thread has enqueued through the library
 * (monotone counter; bench.py reports the difference over the timed region). */
uint64_t vsbp_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* VSBP_H */
