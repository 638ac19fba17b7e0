/*
 * vsbp_oracle.c -- the CPU ORACLE for the stereo hot path of arXiv 1902.09733.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1902_09733_b200/) never links, imports or executes it, and shares no code,
 * header, table or constant with it.
 *
 * Plain, slow, obviously-correct C: scalar loops, no blocking, no fusion, no SIMD,
 * no threads.  Integer BP in int32 fixed point; JBU and reprojection in double.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * DESIGN.md "Readings" R-n = the reading adopted where the paper is silent.
 *
 * Layouts (all row-major, tightly packed, host memory owned by the caller):
 *   images          u8  [H][W]            (grey)      u8 [H][W][3] (RGB)
 *   cost volume D   i32 [H][W][L]
 *   messages M      i32 [4][H][W][L]      M[k][y][x][d] = message pixel (x,y)
 *                                          SENDS toward direction k
 *                                          k: 0 up (y-1), 1 down (y+1),
 *                                             2 left (x-1), 3 right (x+1)
 *   disparity       i32 [H][W] labels;    upsampled: double [sH][sW] full-res px
 *   xyz             double [H][W][3]
 *
 * Error codes: 0 ok, -1 invalid argument, -2 dimension mismatch, -3 overflow.
 *
 * Parity pins for every function: tests/test_oracle_pins.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_EDIM (-2)
#define OR_EOVERFLOW (-3)

/* Fixed-point scale S = 2^7 (R-6): one label of disparity difference
 * costs S in the smoothness term.  Paper: silent on numerics. */
#define ORACLE_FIXED_SHIFT 7

/* ------------------------------------------------------------------------- */
/* O1  parameter quantisation (R-5, R-6, R-7)                        */
/* ------------------------------------------------------------------------- */

/* round half away from zero, evaluated in double */
static int64_t round_half_away(double v)
{
    if (v >= 0.0)
        return (int64_t)floor(v + 0.5);
    return -(int64_t)floor(-v + 0.5);
}

/* out[0] = lambda_q = round(lambda * S)   (weight of the data term, R-5)
 * out[1] = tau_d    = round(data_trunc)   (intensity levels)
 * out[2] = tau_q    = round(disc_trunc*S) (smoothness truncation, fixed point)
 * out[3] = S        = 2^7                 (smoothness slope per label)       */
int oracle_quantize(float lambda, float data_trunc, float disc_trunc, int32_t out[4])
{
    const double S = (double)(1 << ORACLE_FIXED_SHIFT);
    if (!out) return OR_EINVAL;
    if (!(lambda >= 0.0f) || !(data_trunc > 0.0f) || !(disc_trunc > 0.0f)) return OR_EINVAL;
    int64_t lq = round_half_away((double)lambda * S);
    int64_t td = round_half_away((double)data_trunc);
    int64_t tq = round_half_away((double)disc_trunc * S);
    if (td < 1 || tq < 1) return OR_EINVAL;
    if (lq > 0x7fffffff || td > 0x7fffffff || tq > 0x7fffffff) return OR_EOVERFLOW;
    out[0] = (int32_t)lq;
    out[1] = (int32_t)td;
    out[2] = (int32_t)tq;
    out[3] = (int32_t)S;
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O0  prep: RGB -> grey -> s x s box mean  ("downsample the stereo  */
/*     image pairs"; R-22: BT.601 integer grey, area average)      */
/* ------------------------------------------------------------------------- */
int oracle_prep(const uint8_t *rgb, int W_hi, int H_hi, int s, uint8_t *gray_lo)
{
    if (!rgb || !gray_lo || W_hi < 1 || H_hi < 1 || s < 1) return OR_EINVAL;
    if (W_hi % s != 0 || H_hi % s != 0) return OR_EDIM;
    int W = W_hi / s, H = H_hi / s;
    for (int Y = 0; Y < H; ++Y) {
        for (int X = 0; X < W; ++X) {
            int64_t sum = 0;
            for (int j = 0; j < s; ++j) {
                for (int i = 0; i < s; ++i) {
                    const uint8_t *px = rgb + 3 * ((size_t)(Y * s + j) * W_hi + (size_t)(X * s + i));
                    int g = (77 * px[0] + 150 * px[1] + 29 * px[2] + 128) >> 8;
                    sum += g;
                }
            }
            int64_t n = (int64_t)s * s;
            gray_lo[(size_t)Y * W + X] = (uint8_t)((sum + n / 2) / n);
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O2  data cost E_{D,X}(d)  (Eq.1; R-2 truncated AD, R-8 border)     */
/* D(x,y,d) = lambda_q * min(|L(x,y) - R(x-d,y)|, tau_d)  if x-d >= 0          */
/*          = lambda_q * tau_d                             otherwise           */
/* ------------------------------------------------------------------------- */
int oracle_cost_volume(const uint8_t *left, const uint8_t *right, int W, int H, int L,
                       int32_t lam_q, int32_t tau_d, int32_t *D)
{
    if (!left || !right || !D || W < 1 || H < 1 || L < 2 || lam_q < 0 || tau_d < 1) return OR_EINVAL;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int d = 0; d < L; ++d) {
                int32_t c;
                if (x - d >= 0) {
                    int diff = abs((int)left[(size_t)y * W + x] - (int)right[(size_t)y * W + (x - d)]);
                    c = lam_q * (diff < tau_d ? diff : tau_d);
                } else {
                    c = lam_q * tau_d;
                }
                D[((size_t)y * W + x) * L + d] = c;
            }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O3  cost pyramid  ("[4]" hierarchical BP; R-12)                        */
/* W' = ceil(W/2), H' = ceil(H/2);  D'(X,Y,d) = sum of D over the existing     */
/* children (2X+i, 2Y+j), i,j in {0,1}.                                        */
/* ------------------------------------------------------------------------- */
int oracle_pyramid_down(const int32_t *D, int W, int H, int L, int32_t *Dn)
{
    if (!D || !Dn || W < 1 || H < 1 || L < 1) return OR_EINVAL;
    int Wn = (W + 1) / 2, Hn = (H + 1) / 2;
    for (int Y = 0; Y < Hn; ++Y)
        for (int X = 0; X < Wn; ++X)
            for (int d = 0; d < L; ++d) {
                int64_t sum = 0;
                for (int j = 0; j < 2; ++j)
                    for (int i = 0; i < 2; ++i) {
                        int x = 2 * X + i, y = 2 * Y + j;
                        if (x < W && y < H) sum += D[((size_t)y * W + x) * L + d];
                    }
                if (sum > 0x7fffffff) return OR_EOVERFLOW;
                Dn[((size_t)Y * Wn + X) * L + d] = (int32_t)sum;
            }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O4  one message  (Eq.1 "M_{Y,X}(d) is the message vector passed     */
/* from a pixel to its neighbor"; R-3 truncated linear smoothness, R-9 min-    */
/* normalisation; S:137-145, S:168 two-pass O(L) distance transform)           */
/*                                                                             */
/*   m(d) = min( min_{d'} h(d') + S*|d-d'| ,  min_{d'} h(d') + tau_q ) - min h */
/*                                                                             */
/* The inner min over d' is the lower envelope of cones computed by the two-   */
/* pass distance transform: f(d) = min(h(d), f(d-1)+S) forward, then           */
/* g(d) = min(f(d), g(d+1)+S) backward.                                        */
/* ------------------------------------------------------------------------- */
int oracle_message(const int32_t *h, int L, int32_t S, int32_t tau_q, int32_t *m)
{
    if (!h || !m || L < 1 || S < 0 || tau_q < 0) return OR_EINVAL;
    int32_t *g = (int32_t *)malloc(sizeof(int32_t) * (size_t)L);
    if (!g) return OR_EINVAL;
    /* forward pass */
    g[0] = h[0];
    for (int d = 1; d < L; ++d) {
        int32_t a = h[d], b = g[d - 1] + S;
        g[d] = a < b ? a : b;
    }
    /* backward pass */
    for (int d = L - 2; d >= 0; --d) {
        int32_t b = g[d + 1] + S;
        if (b < g[d]) g[d] = b;
    }
    int32_t hmin = h[0];
    for (int d = 1; d < L; ++d)
        if (h[d] < hmin) hmin = h[d];
    for (int d = 0; d < L; ++d) {
        int32_t t = hmin + tau_q;
        int32_t v = g[d] < t ? g[d] : t;
        m[d] = v - hmin;
    }
    free(g);
    return OR_OK;
}

/* neighbour of (x,y) in direction k; returns 0 if it does not exist */
static int neighbour(int x, int y, int k, int W, int H, int *nx, int *ny)
{
    static const int dx[4] = {0, 0, -1, 1};
    static const int dy[4] = {-1, 1, 0, 0};
    int qx = x + dx[k], qy = y + dy[k];
    if (qx < 0 || qy < 0 || qx >= W || qy >= H) return 0;
    *nx = qx;
    *ny = qy;
    return 1;
}

/* the direction in which neighbour q (lying in direction k of p) sends back to p */
static int opposite(int k)
{
    static const int opp[4] = {1, 0, 3, 2};
    return opp[k];
}

#define MSG(M, k, x, y, W, H, L) ((M) + ((((size_t)(k) * (H) + (y)) * (W) + (x)) * (L)))

/* incoming message to p=(x,y) from its neighbour in direction k (0 if none),
 * copied into in[0..L) */
static void incoming(const int32_t *M, int x, int y, int k, int W, int H, int L, int32_t *in)
{
    int qx, qy;
    if (!neighbour(x, y, k, W, H, &qx, &qy)) {
        for (int d = 0; d < L; ++d) in[d] = 0;
        return;
    }
    const int32_t *src = MSG(M, opposite(k), qx, qy, W, H, L);
    for (int d = 0; d < L; ++d) in[d] = src[d];
}

/* ------------------------------------------------------------------------- */
/* O4  checkerboard BP on one level  (Eq.1, "maximum iteration is */
/* set to 5"; R-10 schedule, R-11 borders)                                     */
/* Iteration t updates every pixel with (x+y+t) mod 2 == 0, in place.  For     */
/* each existing neighbour q (direction k):                                    */
/*   h(d) = D(p,d) + sum_{j != k} in_j(d);  M[k][p] = message(h)               */
/* Messages toward non-existent neighbours are 0 and never computed.           */
/* ------------------------------------------------------------------------- */
int oracle_bp_level(const int32_t *D, int W, int H, int L, int32_t S, int32_t tau_q,
                    int iters, int t0, int32_t *M)
{
    if (!D || !M || W < 1 || H < 1 || L < 1 || iters < 0) return OR_EINVAL;
    int32_t *in = (int32_t *)malloc(sizeof(int32_t) * 4 * (size_t)L);
    int32_t *h = (int32_t *)malloc(sizeof(int32_t) * (size_t)L);
    if (!in || !h) { free(in); free(h); return OR_EINVAL; }
    for (int t = t0; t < t0 + iters; ++t) {
        for (int y = 0; y < H; ++y) {
            for (int x = 0; x < W; ++x) {
                if ((x + y + t) % 2 != 0) continue;
                for (int k = 0; k < 4; ++k) incoming(M, x, y, k, W, H, L, in + (size_t)k * L);
                for (int k = 0; k < 4; ++k) {
                    int qx, qy;
                    int32_t *out = MSG(M, k, x, y, W, H, L);
                    if (!neighbour(x, y, k, W, H, &qx, &qy)) {
                        for (int d = 0; d < L; ++d) out[d] = 0;
                        continue;
                    }
                    for (int d = 0; d < L; ++d) {
                        int32_t v = D[((size_t)y * W + x) * L + d];
                        for (int j = 0; j < 4; ++j)
                            if (j != k) v += in[(size_t)j * L + d];
                        h[d] = v;
                    }
                    oracle_message(h, L, S, tau_q, out);
                }
            }
        }
    }
    free(in);
    free(h);
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O4  message initialisation of level l from level l+1 (R-12):                */
/*   m^l_{p,k} = m^{l+1}_{P(p),k}  if p has a neighbour in direction k, else 0 */
/*   P(x,y) = (floor(x/2), floor(y/2)).                                        */
/* ------------------------------------------------------------------------- */
int oracle_upcopy(const int32_t *Mp, int Wp, int Hp, int W, int H, int L, int32_t *M)
{
    if (!Mp || !M || W < 1 || H < 1 || L < 1) return OR_EINVAL;
    if (Wp != (W + 1) / 2 || Hp != (H + 1) / 2) return OR_EDIM;
    for (int k = 0; k < 4; ++k)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                int qx, qy;
                int32_t *dst = MSG(M, k, x, y, W, H, L);
                if (!neighbour(x, y, k, W, H, &qx, &qy)) {
                    for (int d = 0; d < L; ++d) dst[d] = 0;
                    continue;
                }
                const int32_t *src = MSG(Mp, k, x / 2, y / 2, Wp, Hp, L);
                for (int d = 0; d < L; ++d) dst[d] = src[d];
            }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O6  WTA  ("the label d that minimizes E_X(d) is assigned to each pixel"; */
/* Eq.1 E_X(d) = E_D,X(d) + sum_{Y in N(X)} M_{Y,X}(d); R-13 ties -> smallest d) */
/* ------------------------------------------------------------------------- */
int oracle_wta(const int32_t *D, const int32_t *M, int W, int H, int L, int32_t *disp)
{
    if (!D || !M || !disp || W < 1 || H < 1 || L < 1) return OR_EINVAL;
    int32_t *in = (int32_t *)malloc(sizeof(int32_t) * 4 * (size_t)L);
    if (!in) return OR_EINVAL;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            for (int k = 0; k < 4; ++k) incoming(M, x, y, k, W, H, L, in + (size_t)k * L);
            int best = 0;
            int64_t bestv = 0;
            for (int d = 0; d < L; ++d) {
                int64_t e = D[((size_t)y * W + x) * L + d];
                for (int k = 0; k < 4; ++k) e += in[(size_t)k * L + d];
                if (d == 0 || e < bestv) { bestv = e; best = d; }
            }
            disp[(size_t)y * W + x] = best;
        }
    free(in);
    return OR_OK;
}

/* number of int32 entries of the per-level message fields, all levels */
static size_t level_dims(int W, int H, int levels, int *Ws, int *Hs)
{
    size_t total = 0;
    int w = W, h = H;
    for (int l = 0; l < levels; ++l) {
        Ws[l] = w;
        Hs[l] = h;
        total += (size_t)w * h;
        w = (w + 1) / 2;
        h = (h + 1) / 2;
    }
    return total;
}

/* ------------------------------------------------------------------------- */
/* Full hierarchical BP disparity  ("perform stereo matching on low   */
/* resolution image pairs", "GPU based Belief Propagation [4]", Eq.1, WTA)     */
/*   D_0 = cost volume; D_{l+1} = pyramid(D_l);                                */
/*   top level: M = 0; level l < top: M = upcopy(M_{l+1});                      */
/*   each level: iters checkerboard iterations, t = 0..iters-1;                */
/*   disp = WTA(D_0, M_0).                                                     */
/* msgs_out (optional): all levels' final message fields, level 0 first, each   */
/* [4][H_l][W_l][L] int32.                                                     */
/* ------------------------------------------------------------------------- */
int oracle_bp_disparity(const uint8_t *left, const uint8_t *right, int W, int H, int L,
                        int levels, int iters, float lambda, float data_trunc, float disc_trunc,
                        int32_t *disp, int32_t *msgs_out)
{
    if (!left || !right || !disp || W < 1 || H < 1 || L < 2 || levels < 1 || levels > 16 || iters < 1)
        return OR_EINVAL;
    int32_t q[4];
    int rc = oracle_quantize(lambda, data_trunc, disc_trunc, q);
    if (rc) return rc;
    int32_t lam_q = q[0], tau_d = q[1], tau_q = q[2], S = q[3];
    /* int32 bound (O5, R-25): the largest belief at the top level plus
     * 2^20 of headroom for the distance transform's additions must fit */
    int64_t bound = (int64_t)lam_q * tau_d * ((int64_t)1 << (2 * (levels - 1))) + 4 * (int64_t)tau_q +
                    ((int64_t)1 << 20);
    if (bound >= ((int64_t)1 << 31)) return OR_EOVERFLOW;

    int Ws[16], Hs[16];
    level_dims(W, H, levels, Ws, Hs);
    int32_t *Dl[16] = {0}, *Ml[16] = {0};
    rc = OR_OK;
    for (int l = 0; l < levels; ++l) {
        size_t n = (size_t)Ws[l] * Hs[l] * L;
        Dl[l] = (int32_t *)malloc(sizeof(int32_t) * n);
        Ml[l] = (int32_t *)calloc(4 * n, sizeof(int32_t));
        if (!Dl[l] || !Ml[l]) { rc = OR_EINVAL; goto done; }
    }
    rc = oracle_cost_volume(left, right, W, H, L, lam_q, tau_d, Dl[0]);
    if (rc) goto done;
    for (int l = 0; l + 1 < levels; ++l) {
        rc = oracle_pyramid_down(Dl[l], Ws[l], Hs[l], L, Dl[l + 1]);
        if (rc) goto done;
    }
    for (int l = levels - 1; l >= 0; --l) {
        if (l < levels - 1) {
            rc = oracle_upcopy(Ml[l + 1], Ws[l + 1], Hs[l + 1], Ws[l], Hs[l], L, Ml[l]);
            if (rc) goto done;
        }
        rc = oracle_bp_level(Dl[l], Ws[l], Hs[l], L, S, tau_q, iters, 0, Ml[l]);
        if (rc) goto done;
    }
    rc = oracle_wta(Dl[0], Ml[0], W, H, L, disp);
    if (rc) goto done;
    if (msgs_out) {
        size_t off = 0;
        for (int l = 0; l < levels; ++l) {
            size_t n = 4 * (size_t)Ws[l] * Hs[l] * L;
            memcpy(msgs_out + off, Ml[l], sizeof(int32_t) * n);
            off += n;
        }
    }
done:
    for (int l = 0; l < levels; ++l) { free(Dl[l]); free(Ml[l]); }
    return rc;
}

/* ------------------------------------------------------------------------- */
/* O7  joint bilateral upsampling  (Eq.2; P:84 JBF parameters;          */
/* R-15..R-19)                                                                 */
/*   p = (x,y) full-res; p_down = ((x+0.5)/s - 0.5, (y+0.5)/s - 0.5);           */
/*   window centre c = (floor(x/s), floor(y/s)); taps q in [c-r, c+r]^2 inside  */
/*   the low-res image; I_q = guide at (s*qx + floor(s/2), s*qy + floor(s/2));  */
/*   logit(q) = -|p_down - q|^2/(2 sigma_s^2) - |I_p - I_q|^2/(2 sigma_r^2)     */
/*   (Euclidean RGB distance, 0..255 scale);                                    */
/*   D_p = s * sum_q w_q D'_q / sum_q w_q,  w_q = exp(logit(q) - max_q logit)  */
/* (the max-subtraction cancels in the ratio: it is Eq.2 with K_p = sum w).     */
/* ------------------------------------------------------------------------- */
int oracle_jbu(const int32_t *disp_lo, int W, int H, const uint8_t *guide, int s,
               double sigma_s, double sigma_r, int radius, double *disp_hi)
{
    if (!disp_lo || !guide || !disp_hi || W < 1 || H < 1 || s < 1 || radius < 1) return OR_EINVAL;
    if (!(sigma_s > 0.0) || !(sigma_r > 0.0)) return OR_EINVAL;
    int Wh = W * s, Hh = H * s;
    int ntap = (2 * radius + 1) * (2 * radius + 1);
    double *logit = (double *)malloc(sizeof(double) * (size_t)ntap);
    double *val = (double *)malloc(sizeof(double) * (size_t)ntap);
    if (!logit || !val) { free(logit); free(val); return OR_EINVAL; }
    for (int y = 0; y < Hh; ++y) {
        for (int x = 0; x < Wh; ++x) {
            double px = ((double)x + 0.5) / (double)s - 0.5;
            double py = ((double)y + 0.5) / (double)s - 0.5;
            int cx = x / s, cy = y / s;
            const uint8_t *Ip = guide + 3 * ((size_t)y * Wh + x);
            int n = 0;
            double lmax = -INFINITY;
            for (int qy = cy - radius; qy <= cy + radius; ++qy) {
                for (int qx = cx - radius; qx <= cx + radius; ++qx) {
                    if (qx < 0 || qy < 0 || qx >= W || qy >= H) continue;
                    int gx = s * qx + s / 2, gy = s * qy + s / 2;
                    const uint8_t *Iq = guide + 3 * ((size_t)gy * Wh + gx);
                    double dr = (double)Ip[0] - Iq[0], dg = (double)Ip[1] - Iq[1], db = (double)Ip[2] - Iq[2];
                    double range2 = dr * dr + dg * dg + db * db;
                    double sx = px - qx, sy = py - qy;
                    double spat2 = sx * sx + sy * sy;
                    double l = -spat2 / (2.0 * sigma_s * sigma_s) - range2 / (2.0 * sigma_r * sigma_r);
                    logit[n] = l;
                    val[n] = (double)disp_lo[(size_t)qy * W + qx];
                    if (l > lmax) lmax = l;
                    ++n;
                }
            }
            double num = 0.0, den = 0.0;
            for (int i = 0; i < n; ++i) {
                double w = exp(logit[i] - lmax);
                num += w * val[i];
                den += w;
            }
            disp_hi[(size_t)y * Wh + x] = (double)s * num / den;
        }
    }
    free(logit);
    free(val);
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O8  reprojection  (Eq.3; R-20 z = f*B/(d*du); R-21 min_disp)         */
/*   [X Y Z Wh]^T = Q [u v d 1]^T;  xyz = (X,Y,Z)/Wh if d >= min_disp else NaN  */
/* Q is row-major 4x4.                                                         */
/* ------------------------------------------------------------------------- */
int oracle_reproject(const double *disp, int W, int H, const double *Q, double min_disp,
                     double *xyz, int64_t *n_valid)
{
    if (!disp || !Q || !xyz || !n_valid || W < 1 || H < 1) return OR_EINVAL;
    if (!(min_disp > 0.0)) return OR_EINVAL;
    int64_t count = 0;
    for (int v = 0; v < H; ++v)
        for (int u = 0; u < W; ++u) {
            double d = disp[(size_t)v * W + u];
            double *o = xyz + 3 * ((size_t)v * W + u);
            if (!(d >= min_disp)) {
                o[0] = o[1] = o[2] = NAN;
                continue;
            }
            double in[4] = {(double)u, (double)v, d, 1.0}, out[4];
            for (int r = 0; r < 4; ++r) {
                out[r] = 0.0;
                for (int c = 0; c < 4; ++c) out[r] += Q[4 * r + c] * in[c];
            }
            o[0] = out[0] / out[3];
            o[1] = out[1] / out[3];
            o[2] = out[2] / out[3];
            ++count;
        }
    *n_valid = count;
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* a8  compaction: the pair's point cloud as the list of valid points in raster */
/*     order ("a point cloud"; R-21 validity).  For v = 0..H-1, u = 0..W-1: */
/*     if disp(u,v) >= min_disp, append (X,Y,Z)/Wh of Q [u v d 1]^T (Eq.3).      */
/*     xyz has room for W*H points; *n = the number appended.                   */
/* ------------------------------------------------------------------------- */
int oracle_compact_cloud(const double *disp, int W, int H, const double *Q, double min_disp, double *xyz,
                         int64_t *n)
{
    if (!disp || !Q || !xyz || !n || W < 1 || H < 1) return OR_EINVAL;
    if (!(min_disp > 0.0)) return OR_EINVAL;
    int64_t k = 0;
    for (int v = 0; v < H; ++v)
        for (int u = 0; u < W; ++u) {
            double d = disp[(size_t)v * W + u];
            if (!(d >= min_disp)) continue;
            double in[4] = {(double)u, (double)v, d, 1.0}, out[4];
            for (int r = 0; r < 4; ++r) {
                out[r] = 0.0;
                for (int c = 0; c < 4; ++c) out[r] += Q[4 * r + c] * in[c];
            }
            xyz[3 * k] = out[0] / out[3];
            xyz[3 * k + 1] = out[1] / out[3];
            xyz[3 * k + 2] = out[2] / out[3];
            ++k;
        }
    *n = k;
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* a8  per-pair summary: label sum and an order-independent    */
/* 64-bit hash of the low-res disparity, hash = sum_i mix(i << 32 | label_i)    */
/* mod 2^64, mix = SplitMix64 finaliser.                                       */
/* ------------------------------------------------------------------------- */
static uint64_t oracle_mix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

int oracle_disp_summary(const int32_t *disp, int W, int H, int64_t *label_sum, uint64_t *label_hash)
{
    if (!disp || !label_sum || !label_hash || W < 1 || H < 1) return OR_EINVAL;
    int64_t sum = 0;
    uint64_t hash = 0;
    for (size_t i = 0; i < (size_t)W * H; ++i) {
        sum += disp[i];
        hash += oracle_mix64(((uint64_t)i << 32) | (uint32_t)disp[i]);
    }
    *label_sum = sum;
    *label_hash = hash;
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* F1  rectification: undistortion map + bilinear remap  (§2.1: "only     */
/*     radial distortion and does not have any tangential distortion";         */
/*     "rectify and undistort individual images ... cvInitUndistortMap() and   */
/*     cvRemap()"; R-26, R-27)                          */
/* ------------------------------------------------------------------------- */

/* Destination -> source map ("maps are built destination->source"),
 * cam = {f_u, f_v, c_u, c_v, k1, k2, k3}, new camera matrix = old (no extrinsic
 * rectification for virtual pairs).  For destination pixel (u, v):
 *   x = (u - c_u) / f_u,  y = (v - c_v) / f_v,  r2 = x*x + y*y
 *   kr = 1 + k1*r2 + k2*r2*r2 + k3*r2*r2*r2          (radial only)
 *   src_u = f_u*x*kr + c_u,  src_v = f_v*y*kr + c_v
 * evaluated in double, left to right as written, then quantised to 1/32 px
 * (R-26: the 5 fractional bits of OpenCV's remap tables):
 *   map = floor(src * 32 + 0.5).                                              */
int oracle_undistort_map(int W, int H, const double *cam, int32_t *map_x, int32_t *map_y)
{
    if (W < 1 || H < 1 || !cam || !map_x || !map_y) return OR_EINVAL;
    const double fu = cam[0], fv = cam[1], cu = cam[2], cv = cam[3];
    const double k1 = cam[4], k2 = cam[5], k3 = cam[6];
    if (!(fu > 0.0) || !(fv > 0.0)) return OR_EINVAL;
    /* domain (R-26): |source coordinate| < 2^24 px everywhere, by the bound
     * |src| <= f*max|x|*(1 + |k1| r2m + |k2| r2m^2 + |k3| r2m^3) + |c| with the
     * corner maxima max|x|, max|y|, r2m = max|x|^2 + max|y|^2 */
    {
        double xm = fmax(fabs((0.0 - cu) / fu), fabs(((double)(W - 1) - cu) / fu));
        double ym = fmax(fabs((0.0 - cv) / fv), fabs(((double)(H - 1) - cv) / fv));
        double r2m = xm * xm + ym * ym;
        double K = 1.0 + fabs(k1) * r2m + fabs(k2) * r2m * r2m + fabs(k3) * r2m * r2m * r2m;
        if (!(fu * xm * K + fabs(cu) < 16777216.0) || !(fv * ym * K + fabs(cv) < 16777216.0)) return OR_EOVERFLOW;
    }
    for (int v = 0; v < H; ++v) {
        for (int u = 0; u < W; ++u) {
            double x = ((double)u - cu) / fu;
            double y = ((double)v - cv) / fv;
            double r2 = x * x + y * y;
            double kr = 1.0 + k1 * r2 + k2 * r2 * r2 + k3 * r2 * r2 * r2;
            double su = fu * x * kr + cu;
            double sv = fv * y * kr + cv;
            double qx = floor(su * 32.0 + 0.5), qy = floor(sv * 32.0 + 0.5);
            map_x[(size_t)v * W + u] = (int32_t)qx;
            map_y[(size_t)v * W + u] = (int32_t)qy;
        }
    }
    return OR_OK;
}

/* floor(a / 32) for any int32 a */
static int32_t floor_div32(int32_t a)
{
    return a >= 0 ? a / 32 : -((-(int64_t)a + 31) / 32);
}

/* Bilinear remap of an RGB image through a 1/32-px map (cvRemap, INTER_LINEAR,
 * BORDER_CONSTANT 0; "out-of-bounds sources produce 0").  R-27: integer
 * weights wx = {32 - ax, ax}, wy = {32 - ay, ay} (sum 1024), per channel
 *   out = (sum_{i,j} wx_i * wy_j * I(ix+i, iy+j) + 512) >> 10
 * with I = 0 outside the source image.                                        */
int oracle_remap_rgb(const uint8_t *src, int W, int H, const int32_t *map_x, const int32_t *map_y,
                     uint8_t *dst)
{
    if (!src || !dst || !map_x || !map_y || W < 1 || H < 1) return OR_EINVAL;
    for (int v = 0; v < H; ++v) {
        for (int u = 0; u < W; ++u) {
            int32_t sx = map_x[(size_t)v * W + u], sy = map_y[(size_t)v * W + u];
            int32_t ix = floor_div32(sx), iy = floor_div32(sy);
            int32_t ax = sx - 32 * ix, ay = sy - 32 * iy;
            int32_t wx[2] = {32 - ax, ax}, wy[2] = {32 - ay, ay};
            for (int c = 0; c < 3; ++c) {
                int64_t acc = 0;
                for (int j = 0; j < 2; ++j) {
                    for (int i = 0; i < 2; ++i) {
                        int64_t px = (int64_t)ix + i, py = (int64_t)iy + j;
                        int val = 0;
                        if (px >= 0 && py >= 0 && px < W && py < H) val = src[3 * ((size_t)py * W + (size_t)px) + c];
                        acc += (int64_t)wx[i] * wy[j] * val;
                    }
                }
                dst[3 * ((size_t)v * W + u) + c] = (uint8_t)((acc + 512) >> 10);
            }
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* F3  Harris corners on a grid + ZSSD matching  (§2.3 Eq.4-5; P:84    */
/*     "divide the imaging plane to a 30x30 grid and calculate Harris corners  */
/*     inside each grid individually"; R-28..R-31)    */
/* ------------------------------------------------------------------------- */

/* R-28: Harris response scaled by 25 (k = 0.04 = 1/25), exact in int64.
 *   A = I(x+1,y) - I(x-1,y),  B = I(x,y+1) - I(x,y-1)          (central differences)
 *   Sxx = sum w*A*A, Sxy = sum w*A*B, Syy = sum w*B*B over the 5x5 window with the
 *   binomial weights w(i,j) = b(i) b(j), b = {1,4,6,4,1}     (Eq.4's Gaussian w)
 *   R25 = 25*(Sxx*Syy - Sxy*Sxy) - (Sxx + Syy)^2 = 25 * (det M - k tr^2 M)  (Eq.5)
 * R25 is defined for 3 <= x <= W-4, 3 <= y <= H-4 and set to INT64_MIN elsewhere. */
int oracle_harris_response(const uint8_t *img, int W, int H, int64_t *R25)
{
    static const int b[5] = {1, 4, 6, 4, 1};
    if (!img || !R25 || W < 1 || H < 1) return OR_EINVAL;
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            int64_t out = INT64_MIN;
            if (x >= 3 && x <= W - 4 && y >= 3 && y <= H - 4) {
                int64_t sxx = 0, sxy = 0, syy = 0;
                for (int j = -2; j <= 2; ++j) {
                    for (int i = -2; i <= 2; ++i) {
                        int u = x + i, v = y + j;
                        int64_t A = (int64_t)img[(size_t)v * W + u + 1] - img[(size_t)v * W + u - 1];
                        int64_t B = (int64_t)img[(size_t)(v + 1) * W + u] - img[(size_t)(v - 1) * W + u];
                        int64_t w = (int64_t)b[i + 2] * b[j + 2];
                        sxx += w * A * A;
                        sxy += w * A * B;
                        syy += w * B * B;
                    }
                }
                out = 25 * (sxx * syy - sxy * sxy) - (sxx + syy) * (sxx + syy);
            }
            R25[(size_t)y * W + x] = out;
        }
    }
    return OR_OK;
}

/* R-29: corners.  A pixel with 4 <= x <= W-5, 4 <= y <= H-5 is a corner iff
 * R25 >= thr and R25 is strictly greater than all 8 neighbours'.  The
 * image is cut into gc x gr cells, cell (i,j) = [floor(iW/gc), floor((i+1)W/gc)) x
 * [floor(jH/gr), floor((j+1)H/gr)); each cell keeps its K corners of largest R25,
 * ties to raster order (smaller y, then smaller x).  Output slots
 * out[((j*gc + i)*K + rank)] = {x, y} and resp[...] = R25 for rank < count[j*gc+i];
 * unused slots hold {-1, -1} and INT64_MIN.                                    */
int oracle_harris_grid(const int64_t *R25, int W, int H, int gc, int gr, int K, int64_t thr,
                       int32_t *out_xy, int64_t *resp, int32_t *count)
{
    if (!R25 || !out_xy || !resp || !count || W < 1 || H < 1 || gc < 1 || gr < 1 || K < 1 || thr < 1)
        return OR_EINVAL;
    for (int j = 0; j < gr; ++j) {
        for (int i = 0; i < gc; ++i) {
            const int cell = j * gc + i;
            const int x0 = (int)((int64_t)i * W / gc), x1 = (int)((int64_t)(i + 1) * W / gc);
            const int y0 = (int)((int64_t)j * H / gr), y1 = (int)((int64_t)(j + 1) * H / gr);
            int n = 0;
            for (int k = 0; k < K; ++k) {
                out_xy[2 * ((size_t)cell * K + k)] = -1;
                out_xy[2 * ((size_t)cell * K + k) + 1] = -1;
                resp[(size_t)cell * K + k] = INT64_MIN;
            }
            /* raster scan; insertion into the sorted top-K keeps earlier (raster-first)
             * entries ahead of later ones with equal response */
            for (int y = y0; y < y1; ++y) {
                for (int x = x0; x < x1; ++x) {
                    if (x < 4 || x > W - 5 || y < 4 || y > H - 5) continue;
                    int64_t r = R25[(size_t)y * W + x];
                    if (r < thr) continue;
                    int is_max = 1;
                    for (int dy = -1; dy <= 1 && is_max; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (!dx && !dy) continue;
                            if (R25[(size_t)(y + dy) * W + x + dx] >= r) { is_max = 0; break; }
                        }
                    if (!is_max) continue;
                    int pos = n < K ? n : K;
                    while (pos > 0 && resp[(size_t)cell * K + pos - 1] < r) --pos;
                    if (pos >= K) continue;
                    for (int q = (n < K ? n : K - 1); q > pos; --q) {
                        resp[(size_t)cell * K + q] = resp[(size_t)cell * K + q - 1];
                        out_xy[2 * ((size_t)cell * K + q)] = out_xy[2 * ((size_t)cell * K + q - 1)];
                        out_xy[2 * ((size_t)cell * K + q) + 1] = out_xy[2 * ((size_t)cell * K + q - 1) + 1];
                    }
                    resp[(size_t)cell * K + pos] = r;
                    out_xy[2 * ((size_t)cell * K + pos)] = x;
                    out_xy[2 * ((size_t)cell * K + pos) + 1] = y;
                    if (n < K) ++n;
                }
            }
            count[cell] = n;
        }
    }
    return OR_OK;
}

/* R-30: zero-mean SSD ("ZSSD") of the (2r+1)^2 patches of img1 at
 * (x1,y1) and img2 at (x2,y2), scaled by n = (2r+1)^2 to stay an integer:
 *   cost = n * sum (a-b)^2 - (sum a - sum b)^2 = n * ZSSD,
 *   ZSSD = sum ((a - mean a) - (b - mean b))^2.
 * Patches must lie inside their images (else OR_EDIM).                         */
int oracle_zssd(const uint8_t *img1, const uint8_t *img2, int W, int H, int x1, int y1, int x2, int y2, int r,
                int64_t *cost)
{
    if (!img1 || !img2 || !cost || r < 1) return OR_EINVAL;
    if (x1 < r || y1 < r || x1 + r >= W || y1 + r >= H) return OR_EDIM;
    if (x2 < r || y2 < r || x2 + r >= W || y2 + r >= H) return OR_EDIM;
    int64_t n = (int64_t)(2 * r + 1) * (2 * r + 1), sa = 0, sb = 0, sdd = 0;
    for (int j = -r; j <= r; ++j)
        for (int i = -r; i <= r; ++i) {
            int64_t a = img1[(size_t)(y1 + j) * W + x1 + i], bb = img2[(size_t)(y2 + j) * W + x2 + i];
            sa += a;
            sb += bb;
            sdd += (a - bb) * (a - bb);
        }
    *cost = n * sdd - (sa - sb) * (sa - sb);
    return OR_OK;
}

/* R-31: match each corner of img1 into img2: candidates (x+dx, y+dy),
 * |dx|,|dy| <= sr, patch inside img2; best = least cost, ties to raster order of
 * the candidate; accepted iff cost <= max_cost and either no candidate lies at
 * Chebyshev distance > 2 from the best, or 5*second > 6*best with second the least
 * cost among those (the 1.2x ratio gate).  Corners whose img1 patch leaves the
 * image, and unused slots (x < 0), are not matched.
 * match[c] = {x2, y2} or {-1, -1}; mcost[c] = best cost (or -1).               */
int oracle_zssd_match(const uint8_t *img1, const uint8_t *img2, int W, int H, const int32_t *xy, int ncorner,
                      int r, int sr, int64_t max_cost, int32_t *match, int64_t *mcost)
{
    if (!img1 || !img2 || !xy || !match || !mcost || ncorner < 0 || r < 1 || sr < 1 || max_cost < 0) return OR_EINVAL;
    for (int c = 0; c < ncorner; ++c) {
        int x = xy[2 * c], y = xy[2 * c + 1];
        match[2 * c] = match[2 * c + 1] = -1;
        mcost[c] = -1;
        if (x < r || y < r || x + r >= W || y + r >= H) continue;
        int64_t best = INT64_MAX;
        int bx = -1, by = -1;
        for (int v = y - sr; v <= y + sr; ++v)
            for (int u = x - sr; u <= x + sr; ++u) {
                int64_t cst;
                if (oracle_zssd(img1, img2, W, H, x, y, u, v, r, &cst) != OR_OK) continue;
                if (cst < best) { best = cst; bx = u; by = v; }
            }
        if (bx < 0) continue;
        int64_t second = INT64_MAX;
        for (int v = y - sr; v <= y + sr; ++v)
            for (int u = x - sr; u <= x + sr; ++u) {
                int du = u - bx, dv = v - by;
                if (du < 0) du = -du;
                if (dv < 0) dv = -dv;
                if ((du > dv ? du : dv) <= 2) continue;
                int64_t cst;
                if (oracle_zssd(img1, img2, W, H, x, y, u, v, r, &cst) != OR_OK) continue;
                if (cst < second) second = cst;
            }
        int ok = best <= max_cost && (second == INT64_MAX || 5 * second > 6 * best);
        if (ok) {
            match[2 * c] = bx;
            match[2 * c + 1] = by;
            mcost[c] = best;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* F2  constant-space BP  ("GPU based Belief Propagation [4]", [4] = Yang, */
/*     Wang, Ahuja, "A constant-space belief propagation algorithm for stereo   */
/*     matching", CVPR 2010; R-32..R-35)                         */
/*                                                                             */
/* Same energy, quantisation, pyramid dims, checkerboard schedule and border   */
/* rule as the full BP (R-1..R-12), but every pixel of level l keeps only      */
/* k_l = min(L, k0 * 2^l) candidate labels (R-32), with messages over the      */
/* receiver's candidates, stored at the receiver (in[p][k][i] = message p      */
/* receives from its neighbour in direction k, for p's candidate i):           */
/*  * top level T: candidates = the k_T labels of least D_T(p,.), ties to the  */
/*    smaller label; incoming messages 0 (R-33);                               */
/*  * level l < T, parent P = (x/2, y/2): pool = P's candidates; score(d) =    */
/*    D_l(p,d) + sum_k in[P][k][d]; candidates = the k_l pool labels of least  */
/*    score (ties to the smaller label); in[p][k][d] = in[P][k][d] if p has a  */
/*    neighbour in direction k, else 0 (R-34);                                 */
/*  * update of p toward existing neighbour q (direction k), labels c_p, c_q:  */
/*      h(i) = D(p,c_p[i]) + sum_{k' != k} in[p][k'][i]                         */
/*      m(j) = min( min_i h(i) + S |c_p[i] - c_q[j]|, min_i h(i) + tau_q )     */
/*      in[q][opp(k)][j] = m(j) - min_j m(j)                     (R-35)         */
/*  * WTA at level 0: the candidate of least D + sum_k in, ties to the smaller */
/*    label.  Candidate lists are kept in ascending label order.               */
/* D_l is the full-resolution data term summed over the pixel's footprint,    */
/* i.e. the cost pyramid of O3.                                               */
/* ------------------------------------------------------------------------- */

/* indices of the k least values of score[0..n) (ties: smaller key), written in
 * ascending key order (keys ascending in the input) */
static void select_k(const int64_t *score, const int32_t *key, int n, int k, int32_t *out_idx)
{
    char *taken = (char *)calloc((size_t)n, 1);
    int32_t *sel = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
    for (int r = 0; r < k; ++r) {
        int b = -1;
        for (int i = 0; i < n; ++i) {
            if (taken[i]) continue;
            if (b < 0 || score[i] < score[b] || (score[i] == score[b] && key[i] < key[b])) b = i;
        }
        taken[b] = 1;
        sel[r] = b;
    }
    /* ascending key order: keys of the input are ascending, so ascending index */
    int w = 0;
    for (int i = 0; i < n; ++i)
        if (taken[i]) out_idx[w++] = i;
    free(taken);
    free(sel);
}

/* CSBP on a given level-0 data term D0 (i32 [H][W][L], any values >= 0), the
 * quantised smoothness (S, tau_q) given directly.  msg_out (optional): every
 * level's final incoming messages, level 0 first, each [H_l][W_l][4][k_l]
 * (in[p][k][i] as defined above).  Domain: max(D0) * 4^(levels-1) + 4 tau_q +
 * 2^20 < 2^31 (the R-25 bound with max D0 in place of lambda_q tau_d). */
int oracle_csbp_costs(const int32_t *D0, int W, int H, int L, int levels, int iters, int k0, int32_t S,
                      int32_t tau_q, int32_t *disp, int32_t *cand_out, int32_t *msg_out)
{
    if (!D0 || !disp || W < 1 || H < 1 || L < 2 || levels < 1 || levels > 16 || iters < 1 || k0 < 1 || S < 0 ||
        tau_q < 0)
        return OR_EINVAL;
    {
        int64_t dmax = 0;
        for (size_t i = 0; i < (size_t)W * H * L; ++i) {
            if (D0[i] < 0) return OR_EINVAL;
            if (D0[i] > dmax) dmax = D0[i];
        }
        int64_t bound = dmax * ((int64_t)1 << (2 * (levels - 1))) + 4 * (int64_t)tau_q + ((int64_t)1 << 20);
        if (bound >= ((int64_t)1 << 31)) return OR_EOVERFLOW;
    }
    int rc;
    int Ws[16], Hs[16], K[16];
    level_dims(W, H, levels, Ws, Hs);
    for (int l = 0; l < levels; ++l) {
        int64_t k = (int64_t)k0 << l;
        K[l] = k < L ? (int)k : L;
    }
    int32_t *Dl[16] = {0}, *C[16] = {0}, *M[16] = {0};
    rc = OR_OK;
    for (int l = 0; l < levels; ++l) {
        size_t n = (size_t)Ws[l] * Hs[l];
        Dl[l] = (int32_t *)malloc(sizeof(int32_t) * n * L);
        C[l] = (int32_t *)malloc(sizeof(int32_t) * n * K[l]);
        M[l] = (int32_t *)calloc(n * 4 * K[l], sizeof(int32_t));
        if (!Dl[l] || !C[l] || !M[l]) { rc = OR_EINVAL; goto done; }
    }
    memcpy(Dl[0], D0, sizeof(int32_t) * (size_t)W * H * L);
    for (int l = 0; l + 1 < levels; ++l) {
        rc = oracle_pyramid_down(Dl[l], Ws[l], Hs[l], L, Dl[l + 1]);
        if (rc) goto done;
    }
    {
        int64_t *score = (int64_t *)malloc(sizeof(int64_t) * (size_t)L);
        int32_t *keys = (int32_t *)malloc(sizeof(int32_t) * (size_t)L);
        int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)L);
        int64_t *h = (int64_t *)malloc(sizeof(int64_t) * (size_t)L);
        int64_t *m = (int64_t *)malloc(sizeof(int64_t) * (size_t)L);
        for (int l = levels - 1; l >= 0; --l) {
            const int w = Ws[l], hh = Hs[l], k = K[l];
            /* candidates and initial messages (R-33, R-34) */
            for (int y = 0; y < hh; ++y) {
                for (int x = 0; x < w; ++x) {
                    const size_t p = (size_t)y * w + x;
                    int32_t *cp = C[l] + p * k;
                    int32_t *mp = M[l] + p * 4 * k;
                    const int32_t *Dp = Dl[l] + p * L;
                    if (l == levels - 1) {
                        for (int d = 0; d < L; ++d) {
                            score[d] = Dp[d];
                            keys[d] = d;
                        }
                        select_k(score, keys, L, k, idx);
                        for (int i = 0; i < k; ++i) cp[i] = idx[i];
                        /* messages stay 0 */
                    } else {
                        const int kp = K[l + 1], wp = Ws[l + 1];
                        const size_t P = (size_t)(y / 2) * wp + (x / 2);
                        const int32_t *cP = C[l + 1] + P * kp;
                        const int32_t *mP = M[l + 1] + P * 4 * kp;
                        for (int i = 0; i < kp; ++i) {
                            int64_t s = Dp[cP[i]];
                            for (int kk = 0; kk < 4; ++kk) s += mP[kk * kp + i];
                            score[i] = s;
                            keys[i] = cP[i];
                        }
                        select_k(score, keys, kp, k, idx);
                        for (int i = 0; i < k; ++i) {
                            cp[i] = cP[idx[i]];
                            for (int kk = 0; kk < 4; ++kk) {
                                int nx, ny;
                                mp[kk * k + i] = neighbour(x, y, kk, w, hh, &nx, &ny) ? mP[kk * kp + idx[i]] : 0;
                            }
                        }
                    }
                }
            }
            /* checkerboard iterations (R-10, R-11, R-35) */
            for (int t = 0; t < iters; ++t) {
                for (int y = 0; y < hh; ++y) {
                    for (int x = 0; x < w; ++x) {
                        if (((x + y + t) & 1) != 0) continue;
                        const size_t p = (size_t)y * w + x;
                        const int32_t *cp = C[l] + p * k;
                        const int32_t *mp = M[l] + p * 4 * k;
                        const int32_t *Dp = Dl[l] + p * L;
                        for (int kk = 0; kk < 4; ++kk) {
                            int nx, ny;
                            if (!neighbour(x, y, kk, w, hh, &nx, &ny)) continue;
                            const size_t qq = (size_t)ny * w + nx;
                            const int32_t *cq = C[l] + qq * k;
                            int64_t hmin = INT64_MAX;
                            for (int i = 0; i < k; ++i) {
                                int64_t s = Dp[cp[i]];
                                for (int k2 = 0; k2 < 4; ++k2)
                                    if (k2 != kk) s += mp[k2 * k + i];
                                h[i] = s;
                                if (s < hmin) hmin = s;
                            }
                            int64_t mmin = INT64_MAX;
                            for (int j = 0; j < k; ++j) {
                                int64_t best = hmin + tau_q;
                                for (int i = 0; i < k; ++i) {
                                    int64_t dd = cp[i] - cq[j];
                                    if (dd < 0) dd = -dd;
                                    int64_t v = h[i] + (int64_t)S * dd;
                                    if (v < best) best = v;
                                }
                                m[j] = best;
                                if (best < mmin) mmin = best;
                            }
                            int32_t *dst = M[l] + qq * 4 * k + (size_t)opposite(kk) * k;
                            for (int j = 0; j < k; ++j) dst[j] = (int32_t)(m[j] - mmin);
                        }
                    }
                }
            }
        }
        /* WTA (R-35) */
        for (int y = 0; y < H; ++y) {
            for (int x = 0; x < W; ++x) {
                const size_t p = (size_t)y * W + x;
                const int k = K[0];
                const int32_t *cp = C[0] + p * k;
                const int32_t *mp = M[0] + p * 4 * k;
                int64_t best = INT64_MAX;
                int lab = 0;
                for (int i = 0; i < k; ++i) {
                    int64_t s = Dl[0][p * L + cp[i]];
                    for (int kk = 0; kk < 4; ++kk) s += mp[kk * k + i];
                    if (s < best) { best = s; lab = cp[i]; }  /* ascending labels: first = smaller */
                }
                disp[p] = lab;
            }
        }
        free(score);
        free(keys);
        free(idx);
        free(h);
        free(m);
    }
    if (cand_out) {
        size_t off = 0;
        for (int l = 0; l < levels; ++l) {
            size_t n = (size_t)Ws[l] * Hs[l] * K[l];
            memcpy(cand_out + off, C[l], sizeof(int32_t) * n);
            off += n;
        }
    }
    if (msg_out) {
        size_t off = 0;
        for (int l = 0; l < levels; ++l) {
            size_t n = (size_t)Ws[l] * Hs[l] * 4 * K[l];
            memcpy(msg_out + off, M[l], sizeof(int32_t) * n);
            off += n;
        }
    }
done:
    for (int l = 0; l < levels; ++l) { free(Dl[l]); free(C[l]); free(M[l]); }
    return rc;
}

/* CSBP from the image pair: D0 = the cost volume of O2, then oracle_csbp_costs. */
int oracle_csbp(const uint8_t *left, const uint8_t *right, int W, int H, int L, int levels, int iters, int k0,
                float lambda, float data_trunc, float disc_trunc, int32_t *disp, int32_t *cand_out)
{
    if (!left || !right || !disp || W < 1 || H < 1 || L < 2 || levels < 1 || levels > 16 || iters < 1 || k0 < 1)
        return OR_EINVAL;
    int32_t q[4];
    int rc = oracle_quantize(lambda, data_trunc, disc_trunc, q);
    if (rc) return rc;
    int32_t lam_q = q[0], tau_d = q[1], tau_q = q[2], S = q[3];
    int64_t bound = (int64_t)lam_q * tau_d * ((int64_t)1 << (2 * (levels - 1))) + 4 * (int64_t)tau_q +
                    ((int64_t)1 << 20);
    if (bound >= ((int64_t)1 << 31)) return OR_EOVERFLOW;
    int32_t *D0 = (int32_t *)malloc(sizeof(int32_t) * (size_t)W * H * L);
    if (!D0) return OR_EINVAL;
    rc = oracle_cost_volume(left, right, W, H, L, lam_q, tau_d, D0);
    if (!rc) rc = oracle_csbp_costs(D0, W, H, L, levels, iters, k0, S, tau_q, disp, cand_out, NULL);
    free(D0);
    return rc;
}
