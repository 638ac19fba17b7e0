"""Oracle for row f4 -- point-to-point ICP ("use the CUDA accelerated Iterative
Closest Point (ICP) [6] algorithm to fine-register all point clouds together. We run
ICP on the point clouds calculated from low-resolution disparity maps using
Equation 3"; R-36).  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py): plain numpy in float64, brute-force nearest neighbours, a
library SVD for the rigid update.

Reading R-36 (the paper names the algorithm only):
  points  : float32 xyz clouds; NaN rows (invalid disparities, R-21) are dropped;
            every `stride`-th remaining source point is used (SPEC subsample_stride)
  iterate : T = [R|t] starting at `init`; per iteration
              p = R s + t                 (elementwise, left to right, float64)
              nearest target q of each p by brute force on
              d2 = dx*dx + dy*dy + dz*dz  (ties: smaller target index);
              a pair is kept iff d2 <= max_dist^2
              rms = sqrt(mean kept d2)
              (R_d, t_d) = the least-squares rigid motion of the kept p onto q:
              centroids, H = sum (p - pbar)(q - qbar)^T, SVD H = U S V^T,
              R_d = V diag(1, 1, det(V U^T)) U^T, t_d = qbar - R_d pbar
              T <- (R_d, t_d) o T
            stop after the update when |rms - rms_prev| < eps (converged) or after
            max_iter iterations; no kept pair -> failure (iterations = -1).
"""
from __future__ import annotations

import numpy as np


def _valid(xyz: np.ndarray) -> np.ndarray:
    xyz = np.asarray(xyz, np.float64).reshape(-1, 3)
    return xyz[~np.isnan(xyz).any(axis=1)]


def transform(T: np.ndarray, P: np.ndarray) -> np.ndarray:
    R, t = T[:, :3], T[:, 3]
    out = np.empty_like(P)
    for i in range(3):
        out[:, i] = R[i, 0] * P[:, 0] + R[i, 1] * P[:, 1] + R[i, 2] * P[:, 2] + t[i]
    return out


def nearest(P: np.ndarray, Q: np.ndarray, chunk: int = 2048):
    """Brute force: index and squared distance of the nearest Q row to each P row."""
    idx = np.empty(len(P), np.int64)
    d2 = np.empty(len(P), np.float64)
    for a in range(0, len(P), chunk):
        p = P[a:a + chunk]
        dx = p[:, None, 0] - Q[None, :, 0]
        dy = p[:, None, 1] - Q[None, :, 1]
        dz = p[:, None, 2] - Q[None, :, 2]
        D = dx * dx + dy * dy + dz * dz
        j = np.argmin(D, axis=1)  # first minimum = smaller index
        idx[a:a + chunk] = j
        d2[a:a + chunk] = D[np.arange(len(p)), j]
    return idx, d2


def rigid_update(p: np.ndarray, q: np.ndarray) -> np.ndarray:
    pb, qb = p.mean(axis=0), q.mean(axis=0)
    H = (p - pb).T @ (q - qb)
    U, _, Vt = np.linalg.svd(H)
    V = Vt.T
    Dg = np.diag([1.0, 1.0, np.sign(np.linalg.det(V @ U.T))])
    R = V @ Dg @ U.T
    t = qb - R @ pb
    return np.hstack([R, t[:, None]])


def compose(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """(A o B)(x) = A(B(x))."""
    R = A[:, :3] @ B[:, :3]
    t = A[:, :3] @ B[:, 3] + A[:, 3]
    return np.hstack([R, t[:, None]])


def icp_register(src, tgt, init=None, max_iter: int = 20, max_dist: float = 1.0, eps: float = 1e-4,
                 stride: int = 1):
    """Returns dict(T (3x4), rms, iters, converged, rms_history, n_pairs)."""
    S = _valid(src)[::stride]
    Q = _valid(tgt)
    T = np.hstack([np.eye(3), np.zeros((3, 1))]) if init is None else np.asarray(init, np.float64).reshape(3, 4)
    prev, hist, npairs = np.inf, [], []
    for it in range(1, max_iter + 1):
        P = transform(T, S)
        j, d2 = nearest(P, Q)
        keep = d2 <= max_dist * max_dist
        if not keep.any():
            return dict(T=T, rms=np.nan, iters=-1, converged=False, rms_history=hist, n_pairs=npairs)
        rms = float(np.sqrt(d2[keep].mean()))
        hist.append(rms)
        npairs.append(int(keep.sum()))
        T = compose(rigid_update(P[keep], Q[j[keep]]), T)
        if abs(rms - prev) < eps:
            return dict(T=T, rms=rms, iters=it, converged=True, rms_history=hist, n_pairs=npairs)
        prev = rms
    return dict(T=T, rms=rms, iters=max_iter, converged=False, rms_history=hist, n_pairs=npairs)
