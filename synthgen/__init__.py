"""Seeded synthetic inputs shared by the tests, the oracle and bench.py.

This module holds NONE of the method's arithmetic (no cost, BP, upsampling or
reprojection): it only draws seeded random images and known disparity fields with
the shapes, sizes and structure of the paper's workload:

* 2.7K RGB frames (2704 x 1520, "2.7K resolution") of multi-octave value
  noise plus i.i.d. per-channel noise, so the texture survives a 4x box mean;
* a virtual-stereo right frame ("two frames out of every 10") made by
  forward-warping the left frame by an integer low-res disparity field (a slanted
  ground plane plus axis-aligned "buildings"), larger disparity wins, holes get
  fresh noise;
* small grey pairs for the 64 x 48 configuration: i.i.d. texture shifted by a
  constant or a row-wise plane.
"""
from __future__ import annotations

import numpy as np

FULL_W, FULL_H = 2704, 1520  # 2.7K GoPro frame


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed) & 0xFFFFFFFFFFFFFFFF))


# ----------------------------------------------------------------------------- grey
def iid_gray(seed: int, W: int, H: int, lo: int = 0, hi: int = 256) -> np.ndarray:
    return rng(seed).integers(lo, hi, size=(H, W), dtype=np.uint8)


def shifted_pair(seed: int, W: int, H: int, d0: int):
    """Left = i.i.d. texture; right(x - d0, y) = left(x, y); right's last d0 columns
    are fresh noise.  Truth: disparity d0 at every x >= d0."""
    g = rng(seed)
    left = g.integers(0, 256, size=(H, W), dtype=np.uint8)
    right = g.integers(0, 256, size=(H, W), dtype=np.uint8)
    if d0 < W:
        right[:, : W - d0] = left[:, d0:]
    return left, right


def row_plane_pair(seed: int, W: int, H: int, dmin: int, dmax: int):
    """Row-wise integer plane d(y) = dmin + floor((dmax-dmin+1) * y / H).
    Returns (left, right, d_of_row)."""
    g = rng(seed)
    left = g.integers(0, 256, size=(H, W), dtype=np.uint8)
    right = g.integers(0, 256, size=(H, W), dtype=np.uint8)
    drow = dmin + ((dmax - dmin + 1) * np.arange(H)) // H
    for y in range(H):
        d = int(drow[y])
        if d < W:
            right[y, : W - d] = left[y, d:]
    return left, right, drow.astype(np.int32)


# ----------------------------------------------------------------------------- RGB
def value_noise_rgb(seed: int, W: int, H: int, cells=(64, 32, 16, 8, 4), iid_amp: int = 8) -> np.ndarray:
    """Multi-octave bilinear value noise (cells in full-res px, amplitudes halving)
    plus i.i.d. +-iid_amp per channel; u8 [H][W][3].  Pixel (x, y) samples the
    lattice at ((x+0.5)/c, (y+0.5)/c); the interpolation is separable."""
    g = rng(seed)
    acc = np.zeros((H, W, 3), np.float32)
    amp, total = 1.0, 0.0
    for c in cells:
        gh, gw = H // c + 2, W // c + 2
        lat = g.random((gh, gw, 3), dtype=np.float32)
        xs = (np.arange(W, dtype=np.float32) + 0.5) / c
        x0 = xs.astype(np.int32)
        fx = (xs - x0)[None, :, None]
        A = lat[:, x0] * (1 - fx) + lat[:, x0 + 1] * fx          # (gh, W, 3)
        fy = ((np.arange(c, dtype=np.float32) + 0.5) / c)[None, :, None, None]
        rows = A[:-1, None] * (1 - fy) + A[1:, None] * fy        # (gh-1, c, W, 3)
        acc += amp * rows.reshape(-1, W, 3)[:H]
        total += amp
        amp *= 0.5
    img = acc * (255.0 / total)
    img += g.integers(-iid_amp, iid_amp + 1, size=(H, W, 3), dtype=np.int16).astype(np.float32)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def disparity_field(seed: int, W_lo: int, H_lo: int, dmin: int, dmax: int, n_buildings: int = 4) -> np.ndarray:
    """Integer low-res disparity (labels): slanted ground plane from dmin to
    dmax-12 over the rows, plus n axis-aligned buildings raised by +4..+12."""
    g = rng(seed)
    top = max(dmin, dmax - 12)
    Y = np.arange(H_lo)[:, None]
    d = dmin + ((top - dmin) * Y) // max(H_lo, 1)
    d = np.broadcast_to(d, (H_lo, W_lo)).astype(np.int32).copy()
    for _ in range(n_buildings):
        bw = int(g.integers(max(W_lo // 12, 1), max(W_lo // 4, 2)))
        bh = int(g.integers(max(H_lo // 12, 1), max(H_lo // 4, 2)))
        x0 = int(g.integers(0, max(W_lo - bw, 1)))
        y0 = int(g.integers(0, max(H_lo - bh, 1)))
        d[y0:y0 + bh, x0:x0 + bw] += int(g.integers(4, 13))
    return np.clip(d, dmin, dmax).astype(np.int32)


def forward_warp(left: np.ndarray, d_lo: np.ndarray, s: int, hole_seed: int) -> np.ndarray:
    """right(x - s*d, y) = left(x, y) at full res, larger d wins; holes = fresh noise."""
    H, W = left.shape[:2]
    d_full = np.repeat(np.repeat(d_lo, s, axis=0), s, axis=1)[:H, :W].astype(np.int64)
    ys, xs = np.mgrid[0:H, 0:W]
    xt = xs - s * d_full
    ok = xt >= 0
    zbuf = np.full((H, W), -1, np.int64)
    np.maximum.at(zbuf, (ys[ok], xt[ok]), d_full[ok])
    win = ok.copy()
    win[ok] = zbuf[ys[ok], xt[ok]] == d_full[ok]
    right = rng(hole_seed).integers(0, 256, size=left.shape, dtype=np.uint8)
    right[ys[win], xt[win]] = left[ys[win], xs[win]]
    return right


def stereo_pair_rgb(seed: int, W: int = FULL_W, H: int = FULL_H, s: int = 4, dmin: int = 8, dmax: int = 48):
    """One synthetic virtual-stereo pair: (left RGB, right RGB, d_lo truth labels)."""
    left = value_noise_rgb(seed * 3 + 1, W, H)
    d_lo = disparity_field(seed * 3 + 2, W // s, H // s, dmin, dmax)
    right = forward_warp(left, d_lo, s, seed * 3 + 3)
    return left, right, d_lo


# Synthetic intrinsics for the 2.7K frame (B from P:84)
INTRINSICS = dict(f_du=1400.0, f_dv=1400.0, u0=1351.5, v0=759.5, B=0.5)

# BASELINE.json configurations (the shapes; parity cases and the bench workload)
CONFIGS = {
    1: dict(W=64, H=48, L=16, levels=1, iters=5),
    2: dict(W=676, H=380, L=64, levels=5, iters=5, s=4, dmin=8, dmax=48),
    3: dict(W=676, H=380, L=64, levels=5, iters=5, s=4, dmin=8, dmax=48, radius=2),
    4: dict(W=1352, H=760, L=128, levels=6, iters=8, s=2, dmin=16, dmax=96, radius=3),
}
