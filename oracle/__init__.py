"""CPU oracle for the stereo hot path of arXiv 1902.09733 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product path
(``paper_1902_09733_b200``) never imports, links or executes it; the two share no
code.  The arithmetic lives in ``vsbp_oracle.c`` (plain scalar C, int32 BP, double
JBU / reprojection); this module only marshals numpy arrays through ctypes.

Every function cites the PAPER.md passage it follows (P:n = PAPER.md line n) and
the DESIGN.md reading (R-n) it adopts where the paper is silent.  Pins:
``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vsbp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# VSBP_ORACLE_LIB: load a deliberately MUTATED build of vsbp_oracle.c instead
# (tools/mutation_check.py: proves each pin fails under a plausible mistake)
_LIB_OVERRIDE = os.environ.get("VSBP_ORACLE_LIB")

_ERR = {0: "ok", -1: "EINVAL", -2: "EDIM", -3: "EOVERFLOW"}


class OracleError(RuntimeError):
    def __init__(self, code: int, fn: str):
        super().__init__(f"{fn}: {_ERR.get(code, code)}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no SIMD flags, no fast-math)."""
    if _LIB_OVERRIDE:
        return _LIB_OVERRIDE
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = build()
        L = C.CDLL(path)
        p = C.c_void_p
        i = C.c_int
        f = C.c_float
        dbl = C.c_double
        L.oracle_quantize.argtypes = [f, f, f, p]
        L.oracle_prep.argtypes = [p, i, i, i, p]
        L.oracle_undistort_map.argtypes = [i, i, p, p, p]
        L.oracle_remap_rgb.argtypes = [p, i, i, p, p, p]
        L.oracle_harris_response.argtypes = [p, i, i, p]
        L.oracle_csbp.argtypes = [p, p, i, i, i, i, i, i, f, f, f, p, p]
        L.oracle_csbp_costs.argtypes = [p, i, i, i, i, i, i, C.c_int32, C.c_int32, p, p, p]
        L.oracle_harris_grid.argtypes = [p, i, i, i, i, i, C.c_int64, p, p, p]
        L.oracle_zssd.argtypes = [p, p, i, i, i, i, i, i, i, p]
        L.oracle_zssd_match.argtypes = [p, p, i, i, p, i, i, i, C.c_int64, p, p]
        L.oracle_cost_volume.argtypes = [p, p, i, i, i, C.c_int32, C.c_int32, p]
        L.oracle_pyramid_down.argtypes = [p, i, i, i, p]
        L.oracle_message.argtypes = [p, i, C.c_int32, C.c_int32, p]
        L.oracle_bp_level.argtypes = [p, i, i, i, C.c_int32, C.c_int32, i, i, p]
        L.oracle_upcopy.argtypes = [p, i, i, i, i, i, p]
        L.oracle_wta.argtypes = [p, p, i, i, i, p]
        L.oracle_bp_disparity.argtypes = [p, p, i, i, i, i, i, f, f, f, p, p]
        L.oracle_jbu.argtypes = [p, i, i, p, i, dbl, dbl, i, p]
        L.oracle_reproject.argtypes = [p, i, i, p, dbl, p, p]
        L.oracle_disp_summary.argtypes = [p, i, i, p, p]
        L.oracle_compact_cloud.argtypes = [p, i, i, p, dbl, p, p]
        for name in ("oracle_quantize", "oracle_prep", "oracle_cost_volume", "oracle_pyramid_down",
                     "oracle_message", "oracle_bp_level", "oracle_upcopy", "oracle_wta",
                     "oracle_bp_disparity", "oracle_jbu", "oracle_reproject", "oracle_disp_summary"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def _check(rc: int, fn: str):
    if rc != 0:
        raise OracleError(rc, fn)


# --------------------------------------------------------------------------- params
@dataclass(frozen=True)
class QParams:
    """Quantised BP parameters (R-5..R-7)."""
    lam_q: int
    tau_d: int
    tau_q: int
    S: int


def quantize(lam: float, data_trunc: float, disc_trunc: float) -> QParams:
    out = np.zeros(4, np.int32)
    _check(lib().oracle_quantize(lam, data_trunc, disc_trunc, _ptr(out)), "oracle_quantize")
    return QParams(*[int(v) for v in out])


def level_dims(W: int, H: int, levels: int):
    dims = []
    for _ in range(levels):
        dims.append((W, H))
        W, H = (W + 1) // 2, (H + 1) // 2
    return dims


# --------------------------------------------------------------------------- steps
def prep(rgb: np.ndarray, s: int) -> np.ndarray:
    """a0: RGB u8 [H][W][3] -> grey -> s x s box mean, u8 [H/s][W/s]."""
    rgb = np.ascontiguousarray(rgb, np.uint8)
    H, W, _ = rgb.shape
    out = np.zeros((H // s, W // s), np.uint8)
    _check(lib().oracle_prep(_ptr(rgb), W, H, s, _ptr(out)), "oracle_prep")
    return out


def undistort_map(W: int, H: int, cam) -> tuple[np.ndarray, np.ndarray]:
    """f1 (§2.1 radial-only undistortion, cvInitUndistortMap; R-26):
    destination -> source map in 1/32 px, int32 [H][W] each.
    cam = (f_u, f_v, c_u, c_v, k1, k2, k3)."""
    c = np.ascontiguousarray(np.asarray(cam, np.float64).reshape(7))
    mx = np.zeros((H, W), np.int32)
    my = np.zeros((H, W), np.int32)
    _check(lib().oracle_undistort_map(W, H, _ptr(c), _ptr(mx), _ptr(my)), "oracle_undistort_map")
    return mx, my


def remap_rgb(rgb: np.ndarray, map_x: np.ndarray, map_y: np.ndarray) -> np.ndarray:
    """f1 (P:26 cvRemap; R-27): integer bilinear remap, zero outside."""
    rgb = np.ascontiguousarray(rgb, np.uint8)
    H, W, _ = rgb.shape
    mx = np.ascontiguousarray(map_x, np.int32)
    my = np.ascontiguousarray(map_y, np.int32)
    if mx.shape != (H, W) or my.shape != (H, W):
        raise ValueError("map must be [H][W]")
    out = np.zeros_like(rgb)
    _check(lib().oracle_remap_rgb(_ptr(rgb), W, H, _ptr(mx), _ptr(my), _ptr(out)), "oracle_remap_rgb")
    return out


def rectify_prep(rgb: np.ndarray, cam, s: int) -> tuple[np.ndarray, np.ndarray]:
    """f1 + a0: undistort the RGB frame, then grey + s x s box mean.  Returns
    (rectified RGB, grey low-res)."""
    H, W, _ = rgb.shape
    mx, my = undistort_map(W, H, cam)
    rect = remap_rgb(rgb, mx, my)
    return rect, prep(rect, s)


def csbp_k(L: int, levels: int, k0: int) -> list[int]:
    """R-32: candidates per level, k_l = min(L, k0 * 2^l)."""
    return [min(L, k0 << l) for l in range(levels)]


def csbp_disparity(left, right, L, levels, iters, k0, lam=0.07, data_trunc=15.0, disc_trunc=1.7,
                   return_candidates=False):
    """f2 (P:30 [4] = constant-space BP; R-32..R-35): int32 labels [H][W];
    with return_candidates also the per-level candidate lists [H_l][W_l][k_l]."""
    left = np.ascontiguousarray(left, np.uint8)
    right = np.ascontiguousarray(right, np.uint8)
    H, W = left.shape
    disp = np.zeros((H, W), np.int32)
    dims = level_dims(W, H, levels)
    ks = csbp_k(L, levels, k0)
    tot = sum(w * h * k for (w, h), k in zip(dims, ks))
    cand = np.zeros(max(tot, 1), np.int32)
    _check(lib().oracle_csbp(_ptr(left), _ptr(right), W, H, L, levels, iters, k0, lam, data_trunc, disc_trunc,
                             _ptr(disp), _ptr(cand) if return_candidates else None), "oracle_csbp")
    if not return_candidates:
        return disp
    out, off = [], 0
    for (w, h), k in zip(dims, ks):
        out.append(cand[off:off + w * h * k].reshape(h, w, k))
        off += w * h * k
    return disp, out


def csbp_costs(D0: np.ndarray, levels: int, iters: int, k0: int, S: int, tau_q: int):
    """f2 on a given level-0 data term D0 int32 [H][W][L] (R-32..R-35 with the
    smoothness (S, tau_q) given directly).  Returns (disp [H][W], candidates per
    level [H_l][W_l][k_l], final incoming messages per level [H_l][W_l][4][k_l])."""
    D0 = np.ascontiguousarray(D0, np.int32)
    H, W, L = D0.shape
    disp = np.zeros((H, W), np.int32)
    dims = level_dims(W, H, levels)
    ks = csbp_k(L, levels, k0)
    cand = np.zeros(sum(w * h * k for (w, h), k in zip(dims, ks)), np.int32)
    msg = np.zeros(sum(w * h * 4 * k for (w, h), k in zip(dims, ks)), np.int32)
    _check(lib().oracle_csbp_costs(_ptr(D0), W, H, L, levels, iters, k0, S, tau_q, _ptr(disp), _ptr(cand),
                                   _ptr(msg)), "oracle_csbp_costs")
    cands, msgs, oc, om = [], [], 0, 0
    for (w, h), k in zip(dims, ks):
        cands.append(cand[oc:oc + w * h * k].reshape(h, w, k))
        msgs.append(msg[om:om + w * h * 4 * k].reshape(h, w, 4, k))
        oc += w * h * k
        om += w * h * 4 * k
    return disp, cands, msgs


def harris_response(img: np.ndarray) -> np.ndarray:
    """f3 (Eq.4-5; R-28): 25 * Harris response, int64 [H][W]; INT64_MIN
    outside 3 <= x <= W-4, 3 <= y <= H-4."""
    img = np.ascontiguousarray(img, np.uint8)
    H, W = img.shape
    out = np.zeros((H, W), np.int64)
    _check(lib().oracle_harris_response(_ptr(img), W, H, _ptr(out)), "oracle_harris_response")
    return out


def harris_grid(R25: np.ndarray, gc: int = 30, gr: int = 30, K: int = 4, thr: int = 1):
    """f3 (P:84 30x30 grid; R-29): per-cell top-K strict local maxima.  Returns
    (xy int32 [gr*gc*K][2], resp int64 [gr*gc*K], count int32 [gr*gc])."""
    R = np.ascontiguousarray(R25, np.int64)
    H, W = R.shape
    xy = np.zeros((gr * gc * K, 2), np.int32)
    resp = np.zeros(gr * gc * K, np.int64)
    cnt = np.zeros(gr * gc, np.int32)
    _check(lib().oracle_harris_grid(_ptr(R), W, H, gc, gr, K, int(thr), _ptr(xy), _ptr(resp), _ptr(cnt)),
           "oracle_harris_grid")
    return xy, resp, cnt


def zssd(img1, img2, x1, y1, x2, y2, r) -> int:
    """f3 (R-30): n * ZSSD of the n = (2r+1)^2 patches, exact integer."""
    a = np.ascontiguousarray(img1, np.uint8)
    b = np.ascontiguousarray(img2, np.uint8)
    H, W = a.shape
    out = np.zeros(1, np.int64)
    _check(lib().oracle_zssd(_ptr(a), _ptr(b), W, H, x1, y1, x2, y2, r, _ptr(out)), "oracle_zssd")
    return int(out[0])


def zssd_match(img1, img2, xy: np.ndarray, r: int = 5, sr: int = 16, max_cost: int = 2 ** 62):
    """f3 (R-31): best ZSSD match of every corner (slots with x < 0 are
    skipped).  Returns (match int32 [n][2] or -1, cost int64 [n] or -1)."""
    a = np.ascontiguousarray(img1, np.uint8)
    b = np.ascontiguousarray(img2, np.uint8)
    H, W = a.shape
    xy = np.ascontiguousarray(xy, np.int32).reshape(-1, 2)
    n = xy.shape[0]
    m = np.zeros((n, 2), np.int32)
    c = np.zeros(n, np.int64)
    _check(lib().oracle_zssd_match(_ptr(a), _ptr(b), W, H, _ptr(xy), n, r, sr, int(max_cost), _ptr(m), _ptr(c)),
           "oracle_zssd_match")
    return m, c


def cost_volume(left: np.ndarray, right: np.ndarray, L: int, q: QParams) -> np.ndarray:
    """a1 (Eq.1 E_D): int32 [H][W][L]."""
    left = np.ascontiguousarray(left, np.uint8)
    right = np.ascontiguousarray(right, np.uint8)
    H, W = left.shape
    D = np.zeros((H, W, L), np.int32)
    _check(lib().oracle_cost_volume(_ptr(left), _ptr(right), W, H, L, q.lam_q, q.tau_d, _ptr(D)),
           "oracle_cost_volume")
    return D


def pyramid_down(D: np.ndarray) -> np.ndarray:
    """a2 (P:30 [4]): ceil-halved level, sum over existing 2x2 children."""
    D = np.ascontiguousarray(D, np.int32)
    H, W, L = D.shape
    Dn = np.zeros(((H + 1) // 2, (W + 1) // 2, L), np.int32)
    _check(lib().oracle_pyramid_down(_ptr(D), W, H, L, _ptr(Dn)), "oracle_pyramid_down")
    return Dn


def message(h: np.ndarray, S: int, tau_q: int) -> np.ndarray:
    """a4 single message (Eq.1): min(DT_S(h), min h + tau_q) - min h."""
    h = np.ascontiguousarray(h, np.int32)
    m = np.zeros_like(h)
    _check(lib().oracle_message(_ptr(h), h.shape[0], S, tau_q, _ptr(m)), "oracle_message")
    return m


def bp_level(D: np.ndarray, M: np.ndarray, S: int, tau_q: int, iters: int, t0: int = 0) -> np.ndarray:
    """a4: `iters` checkerboard iterations on one level, starting at parity t0.
    M is [4][H][W][L] int32; a new array is returned."""
    D = np.ascontiguousarray(D, np.int32)
    M = np.array(M, np.int32, order="C", copy=True)
    H, W, L = D.shape
    _check(lib().oracle_bp_level(_ptr(D), W, H, L, S, tau_q, iters, t0, _ptr(M)), "oracle_bp_level")
    return M


def upcopy(Mp: np.ndarray, W: int, H: int) -> np.ndarray:
    """a3: child level message init from the parent (R-12)."""
    Mp = np.ascontiguousarray(Mp, np.int32)
    _, Hp, Wp, L = Mp.shape
    M = np.zeros((4, H, W, L), np.int32)
    _check(lib().oracle_upcopy(_ptr(Mp), Wp, Hp, W, H, L, _ptr(M)), "oracle_upcopy")
    return M


def wta(D: np.ndarray, M: np.ndarray) -> np.ndarray:
    """a5: argmin_d D + sum of incoming messages, ties -> smallest d."""
    D = np.ascontiguousarray(D, np.int32)
    M = np.ascontiguousarray(M, np.int32)
    H, W, L = D.shape
    disp = np.zeros((H, W), np.int32)
    _check(lib().oracle_wta(_ptr(D), _ptr(M), W, H, L, _ptr(disp)), "oracle_wta")
    return disp


def bp_disparity(left, right, L, levels, iters, lam=0.07, data_trunc=15.0, disc_trunc=1.7,
                 return_messages=False):
    """a1-a5 end to end: hierarchical checkerboard BP + WTA.
    Returns disp int32 [H][W] (and, optionally, the list of per-level message
    fields [4][H_l][W_l][L], level 0 first)."""
    left = np.ascontiguousarray(left, np.uint8)
    right = np.ascontiguousarray(right, np.uint8)
    H, W = left.shape
    disp = np.zeros((H, W), np.int32)
    dims = level_dims(W, H, levels)
    msgs = None
    if return_messages:
        msgs = np.zeros(sum(4 * w * h * L for w, h in dims), np.int32)
    rc = lib().oracle_bp_disparity(_ptr(left), _ptr(right), W, H, L, levels, iters,
                                   lam, data_trunc, disc_trunc, _ptr(disp),
                                   _ptr(msgs) if msgs is not None else None)
    _check(rc, "oracle_bp_disparity")
    if not return_messages:
        return disp
    out, off = [], 0
    for w, h in dims:
        n = 4 * w * h * L
        out.append(msgs[off:off + n].reshape(4, h, w, L))
        off += n
    return disp, out


def jbu(disp_lo: np.ndarray, guide_rgb: np.ndarray, s: int, sigma_s: float, sigma_r: float,
        radius: int) -> np.ndarray:
    """a6 (Eq.2), double: full-res disparity in full-res pixels."""
    disp_lo = np.ascontiguousarray(disp_lo, np.int32)
    guide_rgb = np.ascontiguousarray(guide_rgb, np.uint8)
    H, W = disp_lo.shape
    assert guide_rgb.shape == (H * s, W * s, 3)
    out = np.zeros((H * s, W * s), np.float64)
    _check(lib().oracle_jbu(_ptr(disp_lo), W, H, _ptr(guide_rgb), s, sigma_s, sigma_r, radius, _ptr(out)),
           "oracle_jbu")
    return out


def reproject(disp: np.ndarray, Q: np.ndarray, min_disp: float = 1.0):
    """a7 (Eq.3), double: xyz [H][W][3] (NaN where d < min_disp), n_valid."""
    disp = np.ascontiguousarray(disp, np.float64)
    Q = np.ascontiguousarray(Q, np.float64).reshape(16)
    H, W = disp.shape
    xyz = np.zeros((H, W, 3), np.float64)
    n = np.zeros(1, np.int64)
    _check(lib().oracle_reproject(_ptr(disp), W, H, _ptr(Q), min_disp, _ptr(xyz), _ptr(n)),
           "oracle_reproject")
    return xyz, int(n[0])


def compact_cloud(disp: np.ndarray, Q: np.ndarray, min_disp: float = 1.0) -> np.ndarray:
    """a8 (R-21): the valid points of Eq.3 in raster order, double [n][3]."""
    disp = np.ascontiguousarray(disp, np.float64)
    Q = np.ascontiguousarray(Q, np.float64).reshape(16)
    H, W = disp.shape
    xyz = np.zeros((H * W, 3), np.float64)
    n = np.zeros(1, np.int64)
    _check(lib().oracle_compact_cloud(_ptr(disp), W, H, _ptr(Q), min_disp, _ptr(xyz), _ptr(n)),
           "oracle_compact_cloud")
    return xyz[: int(n[0])].copy()


def disp_summary(disp: np.ndarray):
    """a8: (label_sum, label_hash) of a low-res disparity map."""
    disp = np.ascontiguousarray(disp, np.int32)
    H, W = disp.shape
    s = np.zeros(1, np.int64)
    h = np.zeros(1, np.uint64)
    _check(lib().oracle_disp_summary(_ptr(disp), W, H, _ptr(s), _ptr(h)), "oracle_disp_summary")
    return int(s[0]), int(h[0])


def q_matrix(f_du: float, f_dv: float, u0: float, v0: float, B: float) -> np.ndarray:
    """Eq.3 as a 4x4 reprojection matrix, z-typo fixed (R-20):
    x = B(u-u0)/d, y = B(v-v0)(f_du/f_dv)/d, z = f_du B/d."""
    return np.array([[1.0, 0.0, 0.0, -u0],
                     [0.0, f_du / f_dv, 0.0, -v0 * f_du / f_dv],
                     [0.0, 0.0, 0.0, f_du],
                     [0.0, 0.0, 1.0 / B, 0.0]], np.float64)


def pipeline_pair(left_rgb, right_rgb, s, L, levels, iters, Q, lam=0.07, data_trunc=15.0,
                  disc_trunc=1.7, sigma_s=None, sigma_r=15.0, radius=None, min_disp=1.0, camera=None):
    """a0-a8 for one pair, the oracle's way (used by bench.py's cpu_baseline);
    with a camera the frames are undistorted first (row f1) and the rectified left
    frame is the JBU guide."""
    if sigma_s is None:
        sigma_s = 15.0 / s
    if radius is None:
        radius = -(-5 // s)
    if camera is not None:
        left_rgb, gl = rectify_prep(left_rgb, camera, s)
        _, gr = rectify_prep(right_rgb, camera, s)
    else:
        gl = prep(left_rgb, s)
        gr = prep(right_rgb, s)
    disp = bp_disparity(gl, gr, L, levels, iters, lam, data_trunc, disc_trunc)
    hi = jbu(disp, left_rgb, s, sigma_s, sigma_r, radius)
    xyz, n = reproject(hi, Q, min_disp)
    return disp, hi, xyz, n
