"""Synthetic UAV video for the C5 stream (BASELINE configs[4]: "stream of 4096
synthetic 2.7K frame pairs"), numpy twin of the device generator synth_video.cu.

Holds NONE of the method's arithmetic.  It renders frames of a camera translating
sideways over a 2.5-D scene, so that consecutive frames form virtual stereo pairs
("two consecutive frames ... a virtual stereo pair", "two frames out of
every 10") and every frame is the right view of one pair and the left view of the
next (S:580-583 with gap = stride):

* world: rows y of the frame, columns X >= 0 of an unbounded strip;
* world disparity (labels, full-res px = s * label):  a ground plane whose label
  depends on the row only, g(y) = dmin + (top - dmin) * (y // s) // (H // s) with
  top = max(dmin, dmax - 12), plus one axis-aligned "building" per world block of
  BW = s * ((W // s) // 2) columns, raised by 4..12 labels;
* texture: 5-octave bilinear value noise (cells 64/32/16/8/4 px, amplitudes
  16/8/4/2/1) + i.i.d. +-8 per channel, attached to the world point;
* frame k, pixel (x, y) sees the world point X with X - k * s * label(X, y) = x
  of largest label (nearer wins); where none exists (a disocclusion) the pixel is
  fresh noise.  Hence right(x - s*d) = left(x) between frames k and k+1 wherever
  the left pixel's world point stays visible.

Everything is integer arithmetic on uint32 hashes (lowbias32), so the CUDA twin
reproduces it bit for bit.
"""
from __future__ import annotations

import numpy as np

M32 = np.uint32(0xFFFFFFFF)
TAG_TEX, TAG_IID, TAG_HOLE, TAG_BLD = 0x7E1, 0x11D, 0x401E, 0xB1D
CELLS = (64, 32, 16, 8, 4)
AMPS = (16, 8, 4, 2, 1)


def hash32(x):
    """lowbias32 (C. Wellons): a 32-bit integer finaliser."""
    x = np.asarray(x, np.uint32)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint32(16))
        x = x * np.uint32(0x7FEB352D)
        x = x ^ (x >> np.uint32(15))
        x = x * np.uint32(0x846CA68B)
        x = x ^ (x >> np.uint32(16))
    return x


def mix(h, v):
    """chain one more value into a hash: hash32(h ^ v)"""
    return hash32(np.asarray(h, np.uint32) ^ np.asarray(v, np.int64).astype(np.uint32))


class VideoScene:
    """The scene and camera path of one synthetic video (seeded)."""

    def __init__(self, seed: int, W: int = 2704, H: int = 1520, s: int = 4, dmin: int = 8, dmax: int = 48):
        if W % s or H % s or dmin < 0 or dmax < dmin:
            raise ValueError("bad video parameters")
        self.seed, self.W, self.H, self.s, self.dmin, self.dmax = int(seed) & 0xFFFFFFFF, W, H, s, dmin, dmax
        self.W_lo, self.H_lo = W // s, H // s
        self.top = max(dmin, dmax - 12)
        self.BW = s * max(self.W_lo // 2, 1)

    # ------------------------------------------------------------------ scene
    def ground(self, y):
        """ground-plane label of full-res row y"""
        return self.dmin + ((self.top - self.dmin) * (np.asarray(y) // self.s)) // self.H_lo

    def building(self, j):
        """building of world block j: (x0, x1, y0, y1) in full-res px (world X
        relative to the block start) and its height in labels (arrays over j)."""
        j = np.asarray(j, np.int64)
        h = mix(hash32(np.uint32(self.seed) ^ np.uint32(TAG_BLD)), j)
        Wb, Hl = self.BW // self.s, self.H_lo
        bw_lo = max(Wb // 6, 1) + (mix(h, 1) % np.uint32(max(Wb // 3, 1))).astype(np.int64)
        bw_lo = np.minimum(bw_lo, Wb)
        bh_lo = max(Hl // 12, 1) + (mix(h, 2) % np.uint32(max(Hl // 6, 1))).astype(np.int64)
        bh_lo = np.minimum(bh_lo, Hl)
        x0 = (mix(h, 3) % np.maximum(Wb - bw_lo + 1, 1).astype(np.uint32)).astype(np.int64)
        y0 = (mix(h, 4) % np.maximum(Hl - bh_lo + 1, 1).astype(np.uint32)).astype(np.int64)
        height = 4 + (mix(h, 5) % np.uint32(9)).astype(np.int64)
        s = self.s
        return s * x0, s * (x0 + bw_lo), s * y0, s * (y0 + bh_lo), height

    def world_label(self, X, y):
        """label of the world surface at (X, y) (X >= 0)"""
        X = np.asarray(X, np.int64)
        y = np.asarray(y, np.int64)
        j = X // self.BW
        x0, x1, y0, y1, height = self.building(j)
        xr = X - j * self.BW
        inside = (xr >= x0) & (xr < x1) & (y >= y0) & (y < y1)
        return self.ground(y) + np.where(inside, height, 0)

    # ------------------------------------------------------------------ texture
    def texture(self, X, y):
        """u8 RGB of world points (X, y): [..., 3]"""
        X = np.asarray(X, np.int64)
        y = np.asarray(y, np.int64)
        out = []
        for ch in range(3):
            hc = mix(hash32(np.uint32(self.seed) ^ np.uint32(TAG_TEX)), ch)
            total = np.zeros(np.broadcast(X, y).shape, np.int64)
            for o, (c, amp) in enumerate(zip(CELLS, AMPS)):
                ho = mix(hc, o)
                lx, fx = X // c, X % c
                ly, fy = y // c, y % c
                wx1, wy1 = 2 * fx + 1, 2 * fy + 1
                wx0, wy0 = 2 * c - wx1, 2 * c - wy1

                def lat(ix, iy):
                    return (mix(mix(ho, ix), iy) & np.uint32(255)).astype(np.int64)

                acc = (lat(lx, ly) * wx0 * wy0 + lat(lx + 1, ly) * wx1 * wy0 +
                       lat(lx, ly + 1) * wx0 * wy1 + lat(lx + 1, ly + 1) * wx1 * wy1)
                total += amp * acc * (4096 // (c * c))
            base = (total + 31 * 8192) // (31 * 16384)
            hi = mix(mix(mix(hash32(np.uint32(self.seed) ^ np.uint32(TAG_IID)), ch), X), y)
            iid = (hi % np.uint32(17)).astype(np.int64) - 8
            out.append(np.clip(base + iid, 0, 255))
        return np.stack(out, axis=-1).astype(np.uint8)

    # ------------------------------------------------------------------ frames
    def visible(self, k: int, rows=None):
        """(label, X) of the world point each full-res pixel of frame k sees;
        label = -1 where none (disocclusion).  rows: optional row subset."""
        ys = np.arange(self.H) if rows is None else np.asarray(rows)
        y = ys[:, None]
        x = np.arange(self.W)[None, :]
        lab = np.full((ys.size, self.W), -1, np.int64)
        Xv = np.zeros((ys.size, self.W), np.int64)
        g = self.ground(y)
        for h in [0] + list(range(4, 13)):  # increasing label: later wins (larger disparity)
            c = g + h
            X = x + k * self.s * c
            ok = self.world_label(X, y) == c
            lab = np.where(ok, c, lab)
            Xv = np.where(ok, X, Xv)
        return lab, Xv

    def frame(self, k: int, rows=None) -> np.ndarray:
        """u8 [H][W][3] frame k (or the given rows)"""
        ys = np.arange(self.H) if rows is None else np.asarray(rows)
        lab, Xv = self.visible(k, ys)
        img = self.texture(Xv, ys[:, None])
        hole = lab < 0
        if hole.any():
            x = np.broadcast_to(np.arange(self.W)[None, :], lab.shape)
            y = np.broadcast_to(ys[:, None], lab.shape)
            hh = mix(mix(hash32(np.uint32(self.seed) ^ np.uint32(TAG_HOLE)), k), x[hole])
            hh = mix(hh, y[hole])
            noise = np.stack([(mix(hh, ch) & np.uint32(255)) for ch in range(3)], axis=-1).astype(np.uint8)
            img[hole] = noise
        return img

    def labels_lo(self, k: int) -> np.ndarray:
        """low-res truth labels of pair k's left view: the label visible at each
        footprint's top-left full-res pixel (-1: hole)"""
        lab, _ = self.visible(k, np.arange(0, self.H, self.s))
        return lab[:, :: self.s].astype(np.int32)


# ----------------------------------------------------------------------------- device twin
_HERE = __import__("os").path.dirname(__import__("os").path.abspath(__file__))
_SYNTH_SRC = __import__("os").path.join(_HERE, "synth_video.cu")
_SYNTH_LIB = __import__("os").path.join(_HERE, "libsynth.so")
_synth = None


def build_device(force: bool = False) -> str:
    """nvcc synth_video.cu -> synthgen/libsynth.so (sm_100a; input generator only)."""
    import os
    import subprocess
    if force or not os.path.exists(_SYNTH_LIB) or os.path.getmtime(_SYNTH_LIB) < os.path.getmtime(_SYNTH_SRC):
        tmp = _SYNTH_LIB + f".tmp{os.getpid()}"
        nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                               "-Xcompiler", "-fPIC", "-o", tmp, _SYNTH_SRC])
        os.replace(tmp, _SYNTH_LIB)
    return _SYNTH_LIB


def _lib():
    global _synth
    if _synth is None:
        import ctypes as C
        L = C.CDLL(build_device())
        L.synth_video_frames.restype = C.c_int
        L.synth_video_frames.argtypes = [C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_void_p, C.c_void_p]
        _synth = L
    return _synth


def frames_device(scene: VideoScene, k0: int, out, stream=None):
    """Render frames k0 .. k0 + out.shape[0] - 1 of `scene` into the CUDA uint8
    tensor out [n][H][W][3] on the device (async on `stream`)."""
    import ctypes as C

    import torch
    n = out.shape[0]
    if tuple(out.shape[1:]) != (scene.H, scene.W, 3) or out.dtype != torch.uint8 or not out.is_cuda \
            or not out.is_contiguous():
        raise ValueError("out must be a contiguous CUDA uint8 [n, H, W, 3] tensor")
    st = torch.cuda.current_stream(out.device) if stream is None else stream
    rc = _lib().synth_video_frames(scene.seed, scene.W, scene.H, scene.s, scene.dmin, scene.dmax, int(k0), n,
                                   C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"synth_video_frames failed ({rc})")
    return out
