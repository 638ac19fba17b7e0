"""Brute-force references that PIN the oracle (DESIGN.md §Oracle pins).

Nothing here re-types the oracle's recurrences: each function computes the same
mathematical object by a different, definitional route --
  * messages by the O(L^2) minimisation over all sender labels (not the two-pass DT),
    normalised by their own minimum (not by min h);
  * exact min-marginals on chains by forward/backward Viterbi;
  * global MAP energies by exhaustive enumeration;
  * synchronous (Jacobi) BP, which the checkerboard schedule must reproduce on the
    colour updated last (textbook bipartite equivalence);
  * Eq.2 literally, without the max-subtraction;
  * Eq.3's forward projection (first line of Eq.3), inverted numerically.
Pure Python / numpy, small sizes only.
"""
from __future__ import annotations

import itertools

import numpy as np

DIRS = [(0, -1), (0, 1), (-1, 0), (1, 0)]  # k: up, down, left, right (dx, dy)
OPP = [1, 0, 3, 2]


def V(a, b, S, tau_q):
    """truncated-linear smoothness (R-3): min(S|a-b|, tau_q)"""
    return np.minimum(S * np.abs(np.subtract.outer(a, b)), tau_q)


def brute_message(h: np.ndarray, S: int, tau_q: int) -> np.ndarray:
    """O(L^2): raw(d) = min_d' h(d') + min(S|d-d'|, tau_q); returned minus min raw."""
    h = np.asarray(h, np.int64)
    L = h.shape[0]
    lab = np.arange(L)
    raw = (h[None, :] + V(lab, lab, S, tau_q)).min(axis=1)  # row d, column d'
    return (raw - raw.min()).astype(np.int64)


def energy(D: np.ndarray, f: np.ndarray, S: int, tau_q: int) -> int:
    """E(f) = sum_p D(p,f_p) + sum_{4-neighbour edges} min(S|f_p - f_q|, tau_q)."""
    H, W, _ = D.shape
    e = int(np.take_along_axis(D, f[..., None].astype(np.int64), axis=2).sum())
    e += int(np.minimum(S * np.abs(np.diff(f.astype(np.int64), axis=1)), tau_q).sum())
    e += int(np.minimum(S * np.abs(np.diff(f.astype(np.int64), axis=0)), tau_q).sum())
    return e


def exhaustive_map(D: np.ndarray, S: int, tau_q: int):
    """Global minimum energy and all minimisers, by enumeration (tiny grids only)."""
    H, W, L = D.shape
    best, arg = None, []
    for lab in itertools.product(range(L), repeat=H * W):
        f = np.array(lab).reshape(H, W)
        e = energy(D, f, S, tau_q)
        if best is None or e < best:
            best, arg = e, [f]
        elif e == best:
            arg.append(f)
    return best, arg


def chain_min_marginals(U: np.ndarray, S: int, tau_q: int) -> np.ndarray:
    """Exact min-marginals mu[x, d] of a chain MRF with unaries U[x, d] (Viterbi
    forward/backward).  mu[x, d] = min over labellings with f_x = d of the energy."""
    U = np.asarray(U, np.int64)
    W, L = U.shape
    lab = np.arange(L)
    Vm = V(lab, lab, S, tau_q)
    a = np.zeros((W, L), np.int64)
    b = np.zeros((W, L), np.int64)
    a[0] = U[0]
    for x in range(1, W):
        a[x] = U[x] + (a[x - 1][:, None] + Vm).min(axis=0)
    b[W - 1] = 0
    for x in range(W - 2, -1, -1):
        b[x] = ((U[x + 1] + b[x + 1])[None, :] + Vm).min(axis=1)
    return a + b


def jacobi_bp(D: np.ndarray, S: int, tau_q: int, T: int) -> np.ndarray:
    """Synchronous BP: every message of step n from the messages of step n-1,
    M^(0) = 0; messages by brute_message.  Returns M^(T) as [4][H][W][L]."""
    H, W, L = D.shape
    M = np.zeros((4, H, W, L), np.int64)
    for _ in range(T):
        Mn = np.zeros_like(M)
        for y in range(H):
            for x in range(W):
                inc = []
                for k, (dx, dy) in enumerate(DIRS):
                    qx, qy = x + dx, y + dy
                    if 0 <= qx < W and 0 <= qy < H:
                        inc.append(M[OPP[k], qy, qx])
                    else:
                        inc.append(np.zeros(L, np.int64))
                for k, (dx, dy) in enumerate(DIRS):
                    qx, qy = x + dx, y + dy
                    if not (0 <= qx < W and 0 <= qy < H):
                        continue
                    h = D[y, x].astype(np.int64) + sum(inc[j] for j in range(4) if j != k)
                    Mn[k, y, x] = brute_message(h, S, tau_q)
        M = Mn
    return M


def beliefs(D: np.ndarray, M: np.ndarray) -> np.ndarray:
    """Eq.1 E_X(d) = E_D,X(d) + sum_{Y in N(X)} M_{Y,X}(d), for every pixel."""
    H, W, L = D.shape
    B = D.astype(np.int64).copy()
    for y in range(H):
        for x in range(W):
            for k, (dx, dy) in enumerate(DIRS):
                qx, qy = x + dx, y + dy
                if 0 <= qx < W and 0 <= qy < H:
                    B[y, x] += M[OPP[k], qy, qx]
    return B


def jbu_literal(disp_lo, guide, s, sigma_s, sigma_r, radius):
    """Eq.2 exactly as printed: D_p = (1/K_p) sum D'_q s(.) g(.), with
    Gaussian s, g, K_p = sum s g; no max-subtraction; returns full-res px (x s)."""
    H, W = disp_lo.shape
    Hh, Wh = H * s, W * s
    out = np.zeros((Hh, Wh))
    for y in range(Hh):
        for x in range(Wh):
            pdx, pdy = (x + 0.5) / s - 0.5, (y + 0.5) / s - 0.5
            cx, cy = x // s, y // s
            Ip = guide[y, x].astype(np.float64)
            num = den = 0.0
            for qy in range(cy - radius, cy + radius + 1):
                for qx in range(cx - radius, cx + radius + 1):
                    if not (0 <= qx < W and 0 <= qy < H):
                        continue
                    Iq = guide[s * qy + s // 2, s * qx + s // 2].astype(np.float64)
                    ws = np.exp(-((pdx - qx) ** 2 + (pdy - qy) ** 2) / (2 * sigma_s ** 2))
                    wr = np.exp(-np.sum((Ip - Iq) ** 2) / (2 * sigma_r ** 2))
                    num += disp_lo[qy, qx] * ws * wr
                    den += ws * wr
            out[y, x] = s * num / den
    return out


def project(xyz, f_du, f_dv, u0, v0, B):
    """Eq.3 first line: [u, v, d] = (1/z)[f x/du, f y/dv, f B/du] + [u0, v0, 0]."""
    x, y, z = xyz
    return f_du * x / z + u0, f_dv * y / z + v0, f_du * B / z
