"""B200-native stereo hot path of arXiv 1902.09733 -- Python binding.

Thin ctypes marshalling over ``libvsbp.so`` (C ABI: ``include/vsbp.h``).  Torch is
used only for device memory and streams; every step of the path runs in the
library's sm_100a kernels.  There is no CPU fallback: if the library is missing
or a call fails, this module raises.

Entry points mirror the C ABI (names follow the paper's steps):
  StereoBP(W, H, ndisp, levels, iters, lam, data_trunc, disc_trunc)  -- bp_create
      .disparity(left, right)                                        -- bp_disparity_batch (a1-a5)
      .messages(pair, level) / .costs(pair, level)                   -- parity exports
  jbu_upsample(disp_lo, guide_rgb, s, sigma_s, sigma_r, radius)      -- a6 (Eq.2)
  reproject(disp, Q, min_disp)                                       -- a7 (Eq.3)
  jbu_reproject(disp_lo, guide_rgb, s, ..., Q, min_disp)             -- a6 + a7 fused
  prep_downsample(rgb, s)                                            -- a0
  pair_summary(disp_lo, n_valid, first_pair_id)                      -- a8
  StereoPipeline                                                     -- a0-a8 for a batch of pairs
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# VSBP_LIB: load another build of the same library (A/B timing experiments in tools/)
LIB_PATH = os.environ.get("VSBP_LIB") or os.path.join(_HERE, "libvsbp.so")

VSBP_OPT_MSG_BYTES = 1
VSBP_OPT_KERNEL = 2
VSBP_OPT_DIMG = 3
VSBP_OPT_FINAL = 4
VSBP_OPT_PAIR = 5
VSBP_OPT_PAIR_BAND = 6
VSBP_OPT_PAIR_MINPX = 7
_ERRNAMES = {-1: "VSBP_EINVAL", -2: "VSBP_EDIM", -3: "VSBP_EOVERFLOW", -4: "VSBP_ECUDA"}


class VsbpError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn}: {_ERRNAMES.get(code, code)} ({msg})")
        self.code = code


_lib = None
_EXPORTS = {
    # name: (restype, argtypes)
    "bp_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_float, C.c_float,
                            C.POINTER(C.c_void_p)]),
    "bp_set_option": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "bp_get_params": (C.c_int, [C.c_void_p, C.c_void_p]),
    "bp_level_dims": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "bp_workspace_bytes": (C.c_size_t, [C.c_void_p, C.c_int]),
    "bp_set_workspace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]),
    "bp_disparity_batch": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "bp_disparity": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "bp_get_messages": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "bp_get_costs": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "bp_destroy": (None, [C.c_void_p]),
    "jbu_upsample_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                     C.c_float, C.c_float, C.c_int, C.c_void_p]),
    "jbu_upsample": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_float,
                               C.c_float, C.c_int, C.c_void_p]),
    "jbu_reproject_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_float,
                                      C.c_float, C.c_int, C.c_void_p, C.c_float, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]),
    "reproject_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_float, C.c_void_p,
                                  C.c_void_p, C.c_void_p]),
    "reproject": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_float, C.c_void_p, C.c_void_p,
                            C.c_void_p]),
    "prep_downsample_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                        C.c_void_p]),
    "prep_downsample": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "icp_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int]),
    "icp_register": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_double,
                               C.c_double, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "csbp_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_float,
                              C.c_float, C.c_void_p]),
    "csbp_workspace_bytes": (C.c_size_t, [C.c_void_p, C.c_int]),
    "csbp_set_workspace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]),
    "csbp_disparity_batch": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "csbp_get_candidates": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "csbp_destroy": (None, [C.c_void_p]),
    "harris_corners_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "zssd_match_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                   C.c_int, C.c_int, C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rectify_prep_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                     C.c_void_p, C.c_void_p]),
    "pair_summary_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_uint64,
                                     C.c_void_p, C.c_void_p]),
    "bp_timing_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "bp_timing_read": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "jbu_timing_enable": (C.c_int, [C.c_int]),
    "jbu_timing_read": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vsbp_q_matrix": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_void_p]),
    "compact_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "compact_cloud_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_float, C.c_void_p,
                                      C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "jbu_compact_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_float, C.c_float,
                                    C.c_int, C.c_void_p, C.c_float, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "vsbp_strerror": (C.c_char_p, [C.c_int]),
    "vsbp_launch_count": (C.c_uint64, []),
}


def lib():
    """Load libvsbp.so (built in-tree by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`. "
                               "There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int, fn: str):
    if rc != 0:
        raise VsbpError(rc, fn, lib().vsbp_strerror(rc).decode())


def _stream(stream=None) -> C.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _dev(t: torch.Tensor, dtype, name: str) -> C.c_void_p:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return C.c_void_p(t.data_ptr())


def launch_count() -> int:
    return int(lib().vsbp_launch_count())


# ----------------------------------------------------------------------------- BP
class StereoBP:
    """Hierarchical checkerboard min-sum BP (Eq.1), a1-a5.  Owns its
    device workspace (a torch uint8 tensor) for up to ``batch`` pairs."""

    def __init__(self, W, H, ndisp, levels, iters, lam=0.07, data_trunc=15.0, disc_trunc=1.7, batch=1,
                 msg_bytes=0, kernel=0, device="cuda", dimg=0, final=None, pair=None, pair_band=None):
        self._h = C.c_void_p()
        _check(lib().bp_create(W, H, ndisp, levels, iters, lam, data_trunc, disc_trunc, C.byref(self._h)),
               "bp_create")
        if msg_bytes:
            _check(lib().bp_set_option(self._h, VSBP_OPT_MSG_BYTES, msg_bytes), "bp_set_option")
        if kernel:
            _check(lib().bp_set_option(self._h, VSBP_OPT_KERNEL, kernel), "bp_set_option")
        if not dimg and os.environ.get("VSBP_DIMG"):  # experiment knob
            dimg = int(os.environ["VSBP_DIMG"])
        if dimg:  # 1: every level-0 update computes D_0 from the images; 2: one-iteration launches only
            _check(lib().bp_set_option(self._h, VSBP_OPT_DIMG, int(dimg)), "bp_set_option")
        if final is None:  # experiment knob: VSBP_FINAL in the environment
            final = int(os.environ.get("VSBP_FINAL", "0"))
        if final:  # fused last level-0 iteration + WTA (level-0 messages not stored)
            _check(lib().bp_set_option(self._h, VSBP_OPT_FINAL, final), "bp_set_option")
        if pair is None:  # experiment knob: VSBP_PAIR=0 disables two iterations per launch
            pair = int(os.environ.get("VSBP_PAIR", "1"))
        _check(lib().bp_set_option(self._h, VSBP_OPT_PAIR, int(pair)), "bp_set_option")
        if pair_band is None and os.environ.get("VSBP_PAIR_BAND"):
            pair_band = int(os.environ["VSBP_PAIR_BAND"])
        if pair_band:
            _check(lib().bp_set_option(self._h, VSBP_OPT_PAIR_BAND, int(pair_band)), "bp_set_option")
        if os.environ.get("VSBP_PAIR_MINPX"):  # experiment knob
            _check(lib().bp_set_option(self._h, VSBP_OPT_PAIR_MINPX, int(os.environ["VSBP_PAIR_MINPX"])),
                   "bp_set_option")
        self.W, self.H, self.L, self.levels, self.iters, self.batch = W, H, ndisp, levels, iters, batch
        nbytes = int(lib().bp_workspace_bytes(self._h, batch))
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _check(lib().bp_set_workspace(self._h, C.c_void_p(self.workspace.data_ptr()), nbytes, batch),
               "bp_set_workspace")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.bp_destroy(h)
            self._h = None

    def params(self) -> dict:
        out = (C.c_int32 * 8)()
        _check(lib().bp_get_params(self._h, out), "bp_get_params")
        keys = ["lam_q", "tau_d", "tau_q", "S", "msg_bytes", "Lp", "levels", "iters"]
        return dict(zip(keys, [int(v) for v in out]))

    def level_dims(self, level: int):
        w, h = C.c_int(), C.c_int()
        _check(lib().bp_level_dims(self._h, level, C.byref(w), C.byref(h)), "bp_level_dims")
        return w.value, h.value

    def disparity(self, left: torch.Tensor, right: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        """left, right: uint8 [B,H,W] (or [H,W]) -> int32 labels of the same shape."""
        squeeze = left.dim() == 2
        if squeeze:
            left, right = left.unsqueeze(0), right.unsqueeze(0)
        B = left.shape[0]
        if tuple(left.shape) != (B, self.H, self.W) or tuple(right.shape) != (B, self.H, self.W):
            raise ValueError(f"expected [B,{self.H},{self.W}] images, got {tuple(left.shape)}, {tuple(right.shape)}")
        if out is None:
            out = torch.empty((B, self.H, self.W), dtype=torch.int32, device=left.device)
        _check(lib().bp_disparity_batch(self._h, B, _dev(left, torch.uint8, "left"),
                                        _dev(right, torch.uint8, "right"), _dev(out, torch.int32, "disp"),
                                        _stream(stream)), "bp_disparity_batch")
        self._last_inputs = (left, right)  # costs(0) may rebuild D_0 from them (VSBP_OPT_DIMG)
        return out[0] if squeeze else out

    def messages(self, pair: int, level: int, stream=None) -> torch.Tensor:
        w, h = self.level_dims(level)
        out = torch.empty((4, h, w, self.L), dtype=torch.int32, device=self.workspace.device)
        _check(lib().bp_get_messages(self._h, pair, level, _dev(out, torch.int32, "out"), _stream(stream)),
               "bp_get_messages")
        return out

    def timing(self, enable: bool = True):
        _check(lib().bp_timing_enable(self._h, 1 if enable else 0), "bp_timing_enable")

    def timing_read(self):
        """Accumulated (since the last read) per-level device ms, launches and
        algorithmic bytes of the message-update kernels."""
        ms = (C.c_double * 16)()
        n = (C.c_int64 * 16)()
        by = (C.c_double * 16)()
        _check(lib().bp_timing_read(self._h, ms, n, by), "bp_timing_read")
        return [dict(level=l, ms=ms[l], launches=int(n[l]), bytes=by[l]) for l in range(self.levels)]

    def costs(self, pair: int, level: int, stream=None) -> torch.Tensor:
        w, h = self.level_dims(level)
        out = torch.empty((h, w, self.L), dtype=torch.int32, device=self.workspace.device)
        _check(lib().bp_get_costs(self._h, pair, level, _dev(out, torch.int32, "out"), _stream(stream)),
               "bp_get_costs")
        return out


class ConstantSpaceBP:
    """Row f2: constant-space BP, the paper's [4] (R-32..R-35).
    Level l keeps k_l = min(ndisp, k0 * 2^l) candidate labels per pixel.  Owns its
    device workspace for up to ``batch`` pairs."""

    def __init__(self, W, H, ndisp, levels, iters, k0, lam=0.07, data_trunc=15.0, disc_trunc=1.7, batch=1,
                 device="cuda"):
        self._h = C.c_void_p()
        _check(lib().csbp_create(W, H, ndisp, levels, iters, k0, lam, data_trunc, disc_trunc, C.byref(self._h)),
               "csbp_create")
        self.W, self.H, self.L, self.levels, self.k0, self.batch = W, H, ndisp, levels, k0, batch
        nbytes = int(lib().csbp_workspace_bytes(self._h, batch))
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _check(lib().csbp_set_workspace(self._h, C.c_void_p(self.workspace.data_ptr()), nbytes, batch),
               "csbp_set_workspace")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.csbp_destroy(h)
            self._h = None

    def k(self, level: int) -> int:
        return min(self.L, self.k0 << level)

    def disparity(self, left: torch.Tensor, right: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        squeeze = left.dim() == 2
        if squeeze:
            left, right = left.unsqueeze(0), right.unsqueeze(0)
        B = left.shape[0]
        if tuple(left.shape) != (B, self.H, self.W) or tuple(right.shape) != (B, self.H, self.W):
            raise ValueError(f"expected [B,{self.H},{self.W}] images")
        if out is None:
            out = torch.empty((B, self.H, self.W), dtype=torch.int32, device=left.device)
        _check(lib().csbp_disparity_batch(self._h, B, _dev(left, torch.uint8, "left"),
                                          _dev(right, torch.uint8, "right"), _dev(out, torch.int32, "disp"),
                                          _stream(stream)), "csbp_disparity_batch")
        return out[0] if squeeze else out

    def candidates(self, pair: int, level: int, stream=None) -> torch.Tensor:
        w, h = self.W, self.H
        for _ in range(level):
            w, h = (w + 1) // 2, (h + 1) // 2
        out = torch.empty((h, w, self.k(level)), dtype=torch.int32, device=self.workspace.device)
        _check(lib().csbp_get_candidates(self._h, pair, level, _dev(out, torch.int32, "out"), _stream(stream)),
               "csbp_get_candidates")
        return out


# ----------------------------------------------------------------------------- a0, a6, a7, a8
def prep_downsample(rgb: torch.Tensor, s: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """rgb: uint8 [n,H,W,3] (or [H,W,3]) -> grey box-downsampled uint8 [n,H/s,W/s]."""
    squeeze = rgb.dim() == 3
    if squeeze:
        rgb = rgb.unsqueeze(0)
    n, H, W, _ = rgb.shape
    if out is None:
        out = torch.empty((n, H // s, W // s), dtype=torch.uint8, device=rgb.device)
    _check(lib().prep_downsample_batch(n, _dev(rgb, torch.uint8, "rgb"), W, H, s, _dev(out, torch.uint8, "gray"),
                                       _stream(stream)), "prep_downsample_batch")
    return out[0] if squeeze else out


def jbu_upsample(disp_lo: torch.Tensor, guide_rgb: torch.Tensor, s: int, sigma_s: float, sigma_r: float,
                 radius: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """disp_lo int32 [B,H,W], guide uint8 [B,sH,sW,3] -> float32 [B,sH,sW] (full-res px)."""
    squeeze = disp_lo.dim() == 2
    if squeeze:
        disp_lo, guide_rgb = disp_lo.unsqueeze(0), guide_rgb.unsqueeze(0)
    B, H, W = disp_lo.shape
    if tuple(guide_rgb.shape) != (B, H * s, W * s, 3):
        raise ValueError("guide must be [B, s*H, s*W, 3]")
    if out is None:
        out = torch.empty((B, H * s, W * s), dtype=torch.float32, device=disp_lo.device)
    _check(lib().jbu_upsample_batch(B, _dev(disp_lo, torch.int32, "disp_lo"), W, H,
                                    _dev(guide_rgb, torch.uint8, "guide_rgb"), s, _dev(out, torch.float32, "disp_hi"),
                                    sigma_s, sigma_r, radius, _stream(stream)), "jbu_upsample_batch")
    return out[0] if squeeze else out


def rectify_prep(rgb_raw: torch.Tensor, cam, s: int, gray: torch.Tensor | None = None,
                 rect: torch.Tensor | bool | None = None, stream=None):
    """Row f1 + a0: undistort (radial k1..k3) and grey/box-downsample n frames.
    rgb_raw uint8 [n,H,W,3] (or [H,W,3]); cam = (f_u, f_v, c_u, c_v, k1, k2, k3).
    rect=True allocates the rectified RGB output (else pass a tensor, or None to
    skip it).  Returns (gray [n,H/s,W/s], rect or None)."""
    squeeze = rgb_raw.dim() == 3
    if squeeze:
        rgb_raw = rgb_raw.unsqueeze(0)
    n, H, W, _ = rgb_raw.shape
    if gray is None:
        gray = torch.empty((n, H // s, W // s), dtype=torch.uint8, device=rgb_raw.device)
    if rect is True:
        rect = torch.empty_like(rgb_raw)
    camd = (C.c_double * 7)(*[float(v) for v in cam])
    _check(lib().rectify_prep_batch(n, _dev(rgb_raw, torch.uint8, "rgb_raw"), W, H, camd, s,
                                    _dev(gray, torch.uint8, "gray_lo"),
                                    _dev(rect, torch.uint8, "rgb_rect") if rect is not None else None,
                                    _stream(stream)), "rectify_prep_batch")
    if squeeze:
        return gray[0], (rect[0] if rect is not None else None)
    return gray, rect


def harris_corners(gray: torch.Tensor, gc: int = 30, gr: int = 30, K: int = 4, thr: int = 10 ** 9, stream=None):
    """Row f3 (Eq.4-5, P:84 30x30 grid): grey uint8 [n,H,W] (or [H,W]) ->
    (R25 int64 [n,H,W], xy int32 [n,gr*gc*K,2], resp int64 [n,gr*gc*K], count int32
    [n,gr*gc]).  R25 = 25 * Harris response (k = 0.04)."""
    squeeze = gray.dim() == 2
    if squeeze:
        gray = gray.unsqueeze(0)
    n, H, W = gray.shape
    d = gray.device
    R25 = torch.empty((n, H, W), dtype=torch.int64, device=d)
    xy = torch.empty((n, gr * gc * K, 2), dtype=torch.int32, device=d)
    resp = torch.empty((n, gr * gc * K), dtype=torch.int64, device=d)
    cnt = torch.empty((n, gr * gc), dtype=torch.int32, device=d)
    _check(lib().harris_corners_batch(n, _dev(gray, torch.uint8, "gray"), W, H, gc, gr, K, int(thr),
                                      _dev(R25, torch.int64, "R25"), _dev(xy, torch.int32, "xy"),
                                      _dev(resp, torch.int64, "resp"), _dev(cnt, torch.int32, "count"),
                                      _stream(stream)), "harris_corners_batch")
    if squeeze:
        return R25[0], xy[0], resp[0], cnt[0]
    return R25, xy, resp, cnt


def zssd_match(img1: torch.Tensor, img2: torch.Tensor, xy: torch.Tensor, r: int = 5, sr: int = 16,
               max_cost: int = 2 ** 62, stream=None):
    """Row f3 (P:56 ZSSD within a search range): corners xy int32 [n,m,2] of img1 ->
    (match int32 [n,m,2] or -1, cost int64 [n,m] = n*ZSSD or -1)."""
    squeeze = img1.dim() == 2
    if squeeze:
        img1, img2, xy = img1.unsqueeze(0), img2.unsqueeze(0), xy.unsqueeze(0)
    n, H, W = img1.shape
    m = xy.shape[1]
    match = torch.empty((n, m, 2), dtype=torch.int32, device=img1.device)
    cost = torch.empty((n, m), dtype=torch.int64, device=img1.device)
    _check(lib().zssd_match_batch(n, _dev(img1, torch.uint8, "img1"), _dev(img2, torch.uint8, "img2"), W, H,
                                  _dev(xy, torch.int32, "xy"), m, r, sr, int(max_cost),
                                  _dev(match, torch.int32, "match"), _dev(cost, torch.int64, "cost"),
                                  _stream(stream)), "zssd_match_batch")
    if squeeze:
        return match[0], cost[0]
    return match, cost


def icp_register(src: torch.Tensor, tgt: torch.Tensor, init=None, max_iter: int = 20, max_dist: float = 1.0,
                 eps: float = 1e-4, stride: int = 1, stream=None) -> torch.Tensor:
    """Row f4 (R-36): point-to-point ICP of float32 [n,3] clouds on the device.
    Returns a device float64 [16] tensor {R|t (12), rms, iterations, converged,
    pairs}; nothing is synchronised."""
    src = src.reshape(-1, 3)
    tgt = tgt.reshape(-1, 3)
    ns, nt = src.shape[0], tgt.shape[0]
    T0 = np.hstack([np.eye(3), np.zeros((3, 1))]) if init is None else np.asarray(init, np.float64).reshape(3, 4)
    initd = (C.c_double * 12)(*[float(v) for v in T0.ravel()])
    nbytes = int(lib().icp_workspace_bytes(ns, nt))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=src.device)
    out = torch.empty(16, dtype=torch.float64, device=src.device)
    _check(lib().icp_register(_dev(src, torch.float32, "src"), ns, _dev(tgt, torch.float32, "tgt"), nt, initd,
                              max_iter, float(max_dist), float(eps), stride, C.c_void_p(ws.data_ptr()), nbytes,
                              _dev(out, torch.float64, "out"), _stream(stream)), "icp_register")
    out._workspace = ws  # keep the workspace alive until the caller is done with `out`
    return out


def q_matrix(f_du: float, f_dv: float, u0: float, v0: float, B: float) -> np.ndarray:
    """Eq.3 as a 4x4 reprojection matrix with z = f B/(d du) (R-20),
    built by the library's vsbp_q_matrix."""
    Q = np.zeros(16, np.float64)
    _check(lib().vsbp_q_matrix(float(f_du), float(f_dv), float(u0), float(v0), float(B),
                               Q.ctypes.data_as(C.c_void_p)), "vsbp_q_matrix")
    return Q.reshape(4, 4)


def reproject(disp: torch.Tensor, Q, min_disp: float = 1.0, xyz: torch.Tensor | None = None,
              n_valid: torch.Tensor | None = None, stream=None):
    """disp float32 [B,H,W] -> (xyz float32 [B,H,W,3], n_valid int64 [B])."""
    squeeze = disp.dim() == 2
    if squeeze:
        disp = disp.unsqueeze(0)
    B, H, W = disp.shape
    Qh = np.ascontiguousarray(np.asarray(Q, np.float64).reshape(16))
    if xyz is None:
        xyz = torch.empty((B, H, W, 3), dtype=torch.float32, device=disp.device)
    if n_valid is None:
        n_valid = torch.empty(B, dtype=torch.int64, device=disp.device)
    _check(lib().reproject_batch(B, _dev(disp, torch.float32, "disp"), W, H, Qh.ctypes.data_as(C.c_void_p),
                                 min_disp, _dev(xyz, torch.float32, "xyz"), _dev(n_valid, torch.int64, "n_valid"),
                                 _stream(stream)), "reproject_batch")
    if squeeze:
        return xyz[0], n_valid
    return xyz, n_valid


def jbu_reproject(disp_lo: torch.Tensor, guide_rgb: torch.Tensor, s: int, sigma_s: float, sigma_r: float,
                  radius: int, Q, min_disp: float = 1.0, disp_hi: torch.Tensor | None = None,
                  xyz: torch.Tensor | None = None, n_valid: torch.Tensor | None = None, stream=None):
    """a6 + a7 fused: -> (disp_hi float32 [B,sH,sW], xyz float32 [B,sH,sW,3], n_valid int64 [B])."""
    if disp_lo.dim() == 2:
        disp_lo, guide_rgb = disp_lo.unsqueeze(0), guide_rgb.unsqueeze(0)
    B, H, W = disp_lo.shape
    if tuple(guide_rgb.shape) != (B, H * s, W * s, 3):
        raise ValueError("guide must be [B, s*H, s*W, 3]")
    dev = disp_lo.device
    if disp_hi is None:
        disp_hi = torch.empty((B, H * s, W * s), dtype=torch.float32, device=dev)
    if xyz is None:
        xyz = torch.empty((B, H * s, W * s, 3), dtype=torch.float32, device=dev)
    if n_valid is None:
        n_valid = torch.empty(B, dtype=torch.int64, device=dev)
    Qh = np.ascontiguousarray(np.asarray(Q, np.float64).reshape(16))
    _check(lib().jbu_reproject_batch(B, _dev(disp_lo, torch.int32, "disp_lo"), W, H,
                                     _dev(guide_rgb, torch.uint8, "guide_rgb"), s, sigma_s, sigma_r, radius,
                                     Qh.ctypes.data_as(C.c_void_p), min_disp, _dev(disp_hi, torch.float32, "disp_hi"),
                                     _dev(xyz, torch.float32, "xyz"), _dev(n_valid, torch.int64, "n_valid"),
                                     _stream(stream)), "jbu_reproject_batch")
    return disp_hi, xyz, n_valid


class CloudCompactor:
    """a8: packed point clouds (compact_cloud_batch).  Owns the look-back workspace
    for batches up to ``batch`` pairs of W x H disparity maps."""

    def __init__(self, W: int, H: int, batch: int, device="cuda"):
        self.W, self.H, self.batch = W, H, batch
        n = int(lib().compact_workspace_bytes(batch, W, H))
        self.workspace = torch.empty(n, dtype=torch.uint8, device=device)

    def __call__(self, disp: torch.Tensor, Q, min_disp: float = 1.0, xyz: torch.Tensor | None = None,
                 offsets: torch.Tensor | None = None, n_valid: torch.Tensor | None = None, stream=None):
        """disp float32 [B,H,W] -> (xyz float32 [cap,3] packed, offsets int64 [B+1], n_valid int64 [B]).
        Pair b's points are xyz[offsets[b]:offsets[b+1]] in raster order."""
        if disp.dim() == 2:
            disp = disp.unsqueeze(0)
        B, H, W = disp.shape
        if (W, H) != (self.W, self.H) or B > self.batch:
            raise ValueError("disparity shape does not match the compactor")
        dev = disp.device
        if xyz is None:
            xyz = torch.empty((B * H * W, 3), dtype=torch.float32, device=dev)
        if offsets is None:
            offsets = torch.empty(B + 1, dtype=torch.int64, device=dev)
        if n_valid is None:
            n_valid = torch.empty(B, dtype=torch.int64, device=dev)
        Qh = np.ascontiguousarray(np.asarray(Q, np.float64).reshape(16))
        _check(lib().compact_cloud_batch(B, _dev(disp, torch.float32, "disp"), W, H, Qh.ctypes.data_as(C.c_void_p),
                                         min_disp, _dev(xyz, torch.float32, "xyz"), xyz.shape[0],
                                         _dev(offsets, torch.int64, "offsets"), _dev(n_valid, torch.int64, "n_valid"),
                                         C.c_void_p(self.workspace.data_ptr()), self.workspace.numel(),
                                         _stream(stream)), "compact_cloud_batch")
        return xyz, offsets, n_valid


def jbu_timing(enable: bool = True):
    """Live CUDA-event timing of the JBU kernel inside every later jbu_compact call
    (include/vsbp.h jbu_timing_enable)."""
    _check(lib().jbu_timing_enable(1 if enable else 0), "jbu_timing_enable")


def jbu_timing_read():
    """{ms, launches, taps} accumulated since the last read (synchronises)."""
    ms, n, taps = C.c_double(), C.c_longlong(), C.c_double()
    _check(lib().jbu_timing_read(C.byref(ms), C.byref(n), C.byref(taps)), "jbu_timing_read")
    return dict(ms=ms.value, launches=int(n.value), taps=taps.value)


def jbu_compact(disp_lo: torch.Tensor, guide_rgb: torch.Tensor, s: int, sigma_s: float, sigma_r: float, radius: int,
                Q, min_disp: float, compactor: CloudCompactor, disp_hi: torch.Tensor | None = None,
                xyz: torch.Tensor | None = None, offsets: torch.Tensor | None = None,
                n_valid: torch.Tensor | None = None, stream=None):
    """a6 + a7 + a8 (jbu_compact_batch): JBU to full res with the compaction's
    count pass folded in, then the packed cloud.  compactor: a CloudCompactor of the
    full-res size (its workspace is used).  Returns (disp_hi, xyz, offsets, n_valid)."""
    if disp_lo.dim() == 2:
        disp_lo, guide_rgb = disp_lo.unsqueeze(0), guide_rgb.unsqueeze(0)
    B, H, W = disp_lo.shape
    if tuple(guide_rgb.shape) != (B, H * s, W * s, 3):
        raise ValueError("guide must be [B, s*H, s*W, 3]")
    if (compactor.W, compactor.H) != (W * s, H * s) or B > compactor.batch:
        raise ValueError("the compactor does not match the output size")
    dev = disp_lo.device
    if disp_hi is None:
        disp_hi = torch.empty((B, H * s, W * s), dtype=torch.float32, device=dev)
    if xyz is None:
        xyz = torch.empty((B * H * s * W * s, 3), dtype=torch.float32, device=dev)
    if offsets is None:
        offsets = torch.empty(B + 1, dtype=torch.int64, device=dev)
    if n_valid is None:
        n_valid = torch.empty(B, dtype=torch.int64, device=dev)
    Qh = np.ascontiguousarray(np.asarray(Q, np.float64).reshape(16))
    _check(lib().jbu_compact_batch(B, _dev(disp_lo, torch.int32, "disp_lo"), W, H,
                                   _dev(guide_rgb, torch.uint8, "guide_rgb"), s, sigma_s, sigma_r, radius,
                                   Qh.ctypes.data_as(C.c_void_p), min_disp, _dev(disp_hi, torch.float32, "disp_hi"),
                                   _dev(xyz, torch.float32, "xyz"), xyz.shape[0], _dev(offsets, torch.int64, "offsets"),
                                   _dev(n_valid, torch.int64, "n_valid"), C.c_void_p(compactor.workspace.data_ptr()),
                                   compactor.workspace.numel(), _stream(stream)), "jbu_compact_batch")
    return disp_hi, xyz, offsets, n_valid


SUMMARY_BYTES = 64


def pair_summary(disp_lo: torch.Tensor, n_valid: torch.Tensor, first_pair_id: int = 0,
                 out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """a8: int64 [B,8] rows {n_valid, label_sum, label_hash (as int64 bits), pair_id, 0,0,0,0}."""
    if disp_lo.dim() == 2:
        disp_lo = disp_lo.unsqueeze(0)
    B, H, W = disp_lo.shape
    if out is None:
        out = torch.empty((B, 8), dtype=torch.int64, device=disp_lo.device)
    _check(lib().pair_summary_batch(B, _dev(disp_lo, torch.int32, "disp_lo"), W, H,
                                    _dev(n_valid, torch.int64, "n_valid"), first_pair_id,
                                    _dev(out, torch.int64, "summary"), _stream(stream)), "pair_summary_batch")
    return out


# ----------------------------------------------------------------------------- a0-a8
class StereoPipeline:
    """The whole hot path for batches of B virtual-stereo pairs of 2.7K RGB frames
    (a0-a8), all on one stream: prep, hierarchical BP, JBU (guide = left frame),
    the point cloud, per-pair summary.  Buffers are allocated once.

    Two input forms:
      * run_frames(frames [B+1,H,W,3]): B+1 consecutive frames of the video, pair j
        = (frame j, frame j+1) -- every frame is the right view of one pair and the
        left view of the next (S:580-583 gap = stride), so it crosses
        the host link and is prepped ONCE;
      * run(left [B,H,W,3], right [B,H,W,3]): independent pairs.
    cloud="packed" (default) writes each pair's valid points in raster order
    (compact_cloud_batch: self.xyz [cap,3], self.offsets [B+1]); cloud="dense"
    writes the NaN-padded [B,H,W,3] cloud of the fused JBU+reprojection kernel."""

    def __init__(self, W_hi, H_hi, s, ndisp, levels, iters, batch, lam=0.07, data_trunc=15.0, disc_trunc=1.7,
                 sigma_s=None, sigma_r=15.0, radius=None, min_disp=1.0, Q=None, device="cuda", msg_bytes=0,
                 camera=None, features=None, csbp_k0=None, cloud="packed"):
        if cloud not in ("packed", "dense"):
            raise ValueError("cloud must be 'packed' or 'dense'")
        self.W_hi, self.H_hi, self.s, self.B = W_hi, H_hi, s, batch
        self.W, self.H = W_hi // s, H_hi // s
        self.sigma_s = 15.0 / s if sigma_s is None else sigma_s  # R-16
        self.sigma_r = sigma_r
        self.radius = -(-5 // s) if radius is None else radius
        self.min_disp = min_disp
        self.Q = Q
        self.cloud = cloud
        if csbp_k0:
            # row f2: the constant-space BP of the paper's [4] in place of the full BP
            self.bp = ConstantSpaceBP(self.W, self.H, ndisp, levels, iters, csbp_k0, lam, data_trunc, disc_trunc,
                                      batch=batch, device=device)
        else:
            # the pipeline never exports messages: the last level-0 iteration and both
            # colours' WTA run as one row-wavefront launch (VSBP_OPT_FINAL = 3); the
            # VSBP_FINAL environment knob still overrides it for experiments
            final = int(os.environ.get("VSBP_FINAL", "3"))
            self.bp = StereoBP(self.W, self.H, ndisp, levels, iters, lam, data_trunc, disc_trunc, batch=batch,
                               msg_bytes=msg_bytes, device=device, final=final)
        dev = torch.device(device)
        # 2B grey frames: [2][B] for independent pairs, the first B+1 for a frame run
        self.gray_flat = torch.empty((2 * batch, self.H, self.W), dtype=torch.uint8, device=dev)
        self.gray = self.gray_flat.view(2, batch, self.H, self.W)
        self.disp = torch.empty((batch, self.H, self.W), dtype=torch.int32, device=dev)
        self.disp_hi = torch.empty((batch, H_hi, W_hi), dtype=torch.float32, device=dev)
        self.n_valid = torch.zeros(batch, dtype=torch.int64, device=dev)
        self.summary = torch.empty((batch, 8), dtype=torch.int64, device=dev)
        if cloud == "packed":
            self.compactor = CloudCompactor(W_hi, H_hi, batch, device=dev)
            self.xyz = torch.empty((batch * H_hi * W_hi, 3), dtype=torch.float32, device=dev)
            self.offsets = torch.zeros(batch + 1, dtype=torch.int64, device=dev)
        else:
            self.xyz = torch.empty((batch, H_hi, W_hi, 3), dtype=torch.float32, device=dev)
            self.offsets = None
        # row f1: with a camera (f_u, f_v, c_u, c_v, k1, k2, k3) the raw frames are
        # undistorted first (fused with a0); the rectified left frame is the JBU guide
        self.camera = camera
        # row f3: features = dict(gc, gr, K, thr, r, sr[, max_cost]) runs Harris on the
        # left grey frame and ZSSD-matches the corners into the right one
        self.features = features
        self.corners = self.matches = None
        self.rect = (torch.empty((batch + 1, H_hi, W_hi, 3), dtype=torch.uint8, device=dev)
                     if camera is not None else None)

    def cloud_of(self, pair: int) -> torch.Tensor:
        """pair j's points of the last run: packed [n_j, 3] rows (raster order), or the
        dense [H, W, 3] map (NaN where invalid)"""
        if self.cloud == "dense":
            return self.xyz[pair]
        o = self.offsets.cpu()
        return self.xyz[int(o[pair]):int(o[pair + 1])]

    # ------------------------------------------------------------------ entry points
    def run(self, left_rgb: torch.Tensor, right_rgb: torch.Tensor, first_pair_id: int = 0, stream=None,
            summary_out: torch.Tensor | None = None):
        """left_rgb, right_rgb: uint8 [B,H_hi,W_hi,3] on the device (independent pairs).
        Returns the per-pair summary tensor (device); disp / disp_hi / xyz stay in the object."""
        guide = self.run_bp(left_rgb, right_rgb, stream)
        return self.run_jbu(guide, first_pair_id, stream, summary_out)

    def run_frames(self, frames: torch.Tensor, first_pair_id: int = 0, stream=None,
                   summary_out: torch.Tensor | None = None):
        """frames: uint8 [n+1,H_hi,W_hi,3] consecutive frames on the device, n <= B:
        the n pairs (frame j, frame j+1).  Every frame is prepped once."""
        n = frames.shape[0] - 1
        if n < 1 or n > self.B:
            raise ValueError(f"need 2..{self.B + 1} frames, got {frames.shape[0]}")
        g = self.gray_flat[:n + 1]
        if self.camera is not None:
            rectify_prep(frames, self.camera, self.s, gray=g, rect=self.rect[:n + 1], stream=stream)
            guide = self.rect[:n]
        else:
            prep_downsample(frames, self.s, out=g, stream=stream)
            guide = frames[:n]
        self._bp_and_features(g[:n], g[1:n + 1], stream)
        return self.run_jbu(guide, first_pair_id, stream, summary_out)

    # ------------------------------------------------------------------ stages
    def run_bp(self, left_rgb: torch.Tensor, right_rgb: torch.Tensor, stream=None) -> torch.Tensor:
        """a0-a5 (and f1/f3 when configured) for independent pairs; returns the JBU guide."""
        B = left_rgb.shape[0]
        if self.camera is not None:
            rectify_prep(left_rgb, self.camera, self.s, gray=self.gray[0, :B], rect=self.rect[:B], stream=stream)
            rectify_prep(right_rgb, self.camera, self.s, gray=self.gray[1, :B], stream=stream)
            guide = self.rect[:B]
        else:
            prep_downsample(left_rgb, self.s, out=self.gray[0, :B], stream=stream)
            prep_downsample(right_rgb, self.s, out=self.gray[1, :B], stream=stream)
            guide = left_rgb
        self._bp_and_features(self.gray[0, :B], self.gray[1, :B], stream)
        return guide

    def _bp_and_features(self, gl: torch.Tensor, gr: torch.Tensor, stream=None):
        B = gl.shape[0]
        self.bp.disparity(gl, gr, out=self.disp[:B], stream=stream)
        if self.features is not None:
            f = self.features
            _, xy, _, _ = harris_corners(gl, f.get("gc", 30), f.get("gr", 30), f.get("K", 4),
                                         f.get("thr", 10 ** 9), stream=stream)
            self.corners = xy
            self.matches = zssd_match(gl, gr, xy, f.get("r", 5), f.get("sr", 16), f.get("max_cost", 2 ** 62),
                                      stream=stream)

    def run_jbu(self, guide: torch.Tensor, first_pair_id: int = 0, stream=None,
                summary_out: torch.Tensor | None = None) -> torch.Tensor:
        """a6-a8 on the labels of the last BP; returns the per-pair summary."""
        B = guide.shape[0]
        if self.cloud == "packed":
            jbu_compact(self.disp[:B], guide, self.s, self.sigma_s, self.sigma_r, self.radius, self.Q, self.min_disp,
                        self.compactor, disp_hi=self.disp_hi[:B], xyz=self.xyz[:B * self.H_hi * self.W_hi],
                        offsets=self.offsets[:B + 1], n_valid=self.n_valid[:B], stream=stream)
        else:
            jbu_reproject(self.disp[:B], guide, self.s, self.sigma_s, self.sigma_r, self.radius, self.Q,
                          self.min_disp, disp_hi=self.disp_hi[:B], xyz=self.xyz[:B], n_valid=self.n_valid[:B],
                          stream=stream)
        out = self.summary[:B] if summary_out is None else summary_out
        return pair_summary(self.disp[:B], self.n_valid[:B], first_pair_id, out=out, stream=stream)


class _HostStream:
    """Stand-in for a CUDA stream / event when the stream plumbing runs on CPU
    tensors (tests with the gloo backend): every operation is already complete."""

    def wait_event(self, ev):
        pass

    def wait_stream(self, st):
        pass

    def record(self, st=None):
        pass

    def query(self):
        return True

    def synchronize(self):
        pass


class StereoStream:
    """End-to-end driver of a video stream (the user-facing call): pinned host frame
    batches in, per-pair summaries (and the device-resident disparity / cloud of the
    last batch) out.

    Batch i is B+1 consecutive frames (pairs first_pair_id + i*pair_stride + j,
    j < B); its host->device copy runs on a copy stream while batch i-1 computes
    (two device slots).  Each batch's summary goes to a ring of device buffers; a
    side stream runs the optional gather (e.g. the NCCL all_gather of the
    summaries) and the device->host copy into a ring of pinned host
    buffers, so neither blocks the compute stream.  on_summary(i, host_tensor) is
    called for EVERY batch, in order, as soon as its copy has landed (polled after
    each enqueue, drained at the end).  Pure stream plumbing: every step of the
    path runs in the library's kernels (StereoPipeline)."""

    def __init__(self, pipeline, device="cuda", ring: int = 4, world: int = 1):
        self.pipe = pipeline
        dev = torch.device(device)
        self.device = dev
        self.cuda = dev.type == "cuda"
        B, Hh, Wh = pipeline.B, pipeline.H_hi, pipeline.W_hi
        self.ring, self.world = ring, world
        self.slots = [torch.empty((B + 1, Hh, Wh, 3), dtype=torch.uint8, device=dev) for _ in range(2)]
        self.sdev = [torch.empty((B, 8), dtype=torch.int64, device=dev) for _ in range(ring)]
        self.gdev = [torch.empty((world * B, 8), dtype=torch.int64, device=dev) for _ in range(ring)]
        pin = self.cuda
        self.host = [torch.empty((world * B, 8), dtype=torch.int64, pin_memory=pin) for _ in range(ring)]
        if self.cuda:
            self.copy_stream = torch.cuda.Stream(device=dev)
            self.side_stream = torch.cuda.Stream(device=dev)
            mk = torch.cuda.Event
        else:
            self.copy_stream = self.side_stream = _HostStream()
            mk = _HostStream
        self.copied = [mk() for _ in range(2)]
        self.freed = [mk() for _ in range(2)]
        self.produced = [mk() for _ in range(ring)]
        self.done = [mk() for _ in range(ring)]
        self.h2d_bytes = self.d2h_bytes = 0

    def _on(self, st):
        import contextlib
        return torch.cuda.stream(st) if self.cuda else contextlib.nullcontext()

    def _compute(self):
        return torch.cuda.current_stream(self.device) if self.cuda else _HostStream()

    def run(self, batches, first_pair_id: int = 0, gather=None, on_summary=None, pair_stride: int | None = None):
        """batches: iterable of pinned host uint8 [n+1,H,W,3] frame batches, n <= B
        (a short batch -- or None / an empty one -- ends a rank's share of the
        stream; every rank must still pass the same number of batches when a
        collective gather is used).  gather(summary [B,8], out [world*B,8]) runs on
        the side stream; rows of missing pairs carry pair id -1 (shard.assemble
        drops them).  Returns the number of batches."""
        from collections import deque
        stride = self.pipe.B if pair_stride is None else pair_stride
        compute = self._compute()
        pending = deque()

        def deliver(block: bool, most: int | None = None):
            """hand finished batches to on_summary in order (block: wait for them)"""
            while pending and (most is None or most > 0) and (block or pending[0][2].query()):
                i, r, ev, rows = pending.popleft()
                ev.synchronize()
                if on_summary is not None:
                    on_summary(i, self.host[r][:rows].clone())
                if most is not None:
                    most -= 1

        n = 0
        B = self.pipe.B
        for i, fh in enumerate(batches):
            k, r = i & 1, i % self.ring
            nf = int(fh.shape[0]) if fh is not None else 0
            npairs = max(nf - 1, 0)  # a short (or empty) batch ends a rank's share of the stream
            dst = self.slots[k][:nf]
            if npairs:
                with self._on(self.copy_stream):
                    if i < 2:
                        self.copy_stream.wait_stream(compute)
                    else:
                        self.copy_stream.wait_event(self.freed[k])
                    dst.copy_(fh, non_blocking=True)
                    self.copied[k].record(self.copy_stream)
                self.h2d_bytes += fh.numel()
            if len(pending) == self.ring:  # ring slot r is still in flight: deliver the oldest first
                deliver(True, 1)
            compute.wait_event(self.done[r])  # the side stream is done with sdev[r] (no-op the first time)
            summ = self.sdev[r]
            if npairs:
                compute.wait_event(self.copied[k])
                self.pipe.run_frames(dst, first_pair_id=first_pair_id + i * stride, summary_out=summ[:npairs])
                self.freed[k].record(compute)
            if npairs < B:
                summ[npairs:].fill_(-1)  # padding rows (pair id -1): every rank gathers B rows
            self.produced[r].record(compute)
            with self._on(self.side_stream):
                self.side_stream.wait_event(self.produced[r])
                if gather is not None:
                    gather(summ, self.gdev[r])
                    src, rows = self.gdev[r], self.world * B
                else:
                    src, rows = summ[:npairs], npairs
                self.host[r][:rows].copy_(src, non_blocking=True)
                self.done[r].record(self.side_stream)
            self.d2h_bytes += rows * 8 * 8
            pending.append((i, r, self.done[r], rows))
            deliver(False)
            n += 1
        deliver(True)
        if self.cuda:
            compute.wait_stream(self.side_stream)
        return n
