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


def jacobi_bp(D: np.ndarray, S: int, tau_q: int, T: int, M0: np.ndarray | None = None) -> np.ndarray:
    """Synchronous BP: every message of step n from the messages of step n-1,
    M^(0) = M0 (default 0); messages by brute_message.  Returns M^(T) as [4][H][W][L]."""
    H, W, L = D.shape
    M = np.zeros((4, H, W, L), np.int64) if M0 is None else np.array(M0, np.int64)
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


# ----------------------------------------------------------------------------- hierarchy
def colour_mask(H: int, W: int, c: int) -> np.ndarray:
    """pixels with (x + y) mod 2 == c"""
    return ((np.arange(H)[:, None] + np.arange(W)[None, :]) % 2) == c


def checkerboard_via_jacobi(D, S, tau_q, T, M0):
    """The state T checkerboard iterations (t = 0..T-1, iteration t updating the
    pixels with (x+y+t) mod 2 == 0) leave, built from SYNCHRONOUS BP started at M0:
    on a bipartite grid the colour updated last, (x+y) mod 2 == (T-1) mod 2, holds
    Jacobi step T and the other colour Jacobi step T-1 (step 0 = M0)."""
    H, W, L = D.shape
    seq = [np.array(M0, np.int64)]
    for _ in range(T):
        seq.append(jacobi_bp(D, S, tau_q, 1, seq[-1]))
    last = colour_mask(H, W, (T - 1) % 2)
    return np.where(last[None, :, :, None], seq[T], seq[T - 1])


def np_cost_volume(left, right, L, lam_q, tau_d):
    """Eq.1's E_D vectorised (R-2, R-8): lam_q * min(|L(x,y) - R(x-d,y)|, tau_d),
    lam_q * tau_d where x - d < 0."""
    left = np.asarray(left, np.int64)
    right = np.asarray(right, np.int64)
    H, W = left.shape
    D = np.full((H, W, L), lam_q * tau_d, np.int64)
    for d in range(min(L, W)):
        D[:, d:, d] = lam_q * np.minimum(np.abs(left[:, d:] - right[:, :W - d]), tau_d)
    return D


def np_pyramid(D):
    """R-12: ceil-halved level = sum over the existing 2x2 children (zero-pad to even, reshape-sum)."""
    H, W, L = D.shape
    P = np.zeros((H + H % 2, W + W % 2, L), np.int64)
    P[:H, :W] = D
    return P.reshape((H + H % 2) // 2, 2, (W + W % 2) // 2, 2, L).sum(axis=(1, 3))


def neighbour_exists(H, W):
    """[4][H][W] bool: pixel (x, y) has a neighbour in direction k (up, down, left, right)."""
    ok = np.ones((4, H, W), bool)
    ok[0, 0, :] = False
    ok[1, H - 1, :] = False
    ok[2, :, 0] = False
    ok[3, :, W - 1] = False
    return ok


def np_upcopy(Mp, W, H):
    """R-12: child (x, y) inherits the parent (x//2, y//2)'s outgoing messages,
    0 toward a missing neighbour (np.repeat, then the edge mask)."""
    M = np.repeat(np.repeat(np.asarray(Mp, np.int64), 2, axis=1), 2, axis=2)[:, :H, :W]
    return np.where(neighbour_exists(H, W)[..., None], M, 0)


def hierarchical_bp(left, right, L, levels, iters, q):
    """Coarse-to-fine BP (P:30 [4]; R-10, R-12) from independent pieces: numpy cost
    volume and pyramid, np.repeat up-copy, each level's checkerboard state from
    synchronous BP started at the up-copied messages (t restarts on every level),
    WTA of the level-0 beliefs (np.argmin: ties -> smallest d).
    Returns (disp, [messages per level, level 0 first])."""
    Ds = [np_cost_volume(left, right, L, q.lam_q, q.tau_d)]
    for _ in range(levels - 1):
        Ds.append(np_pyramid(Ds[-1]))
    Ms = [None] * levels
    for lv in range(levels - 1, -1, -1):
        H, W, _ = Ds[lv].shape
        M0 = np.zeros((4, H, W, L), np.int64) if lv == levels - 1 else np_upcopy(Ms[lv + 1], W, H)
        Ms[lv] = checkerboard_via_jacobi(Ds[lv], q.S, q.tau_q, iters, M0)
    disp = np.argmin(beliefs(Ds[0], Ms[0]), axis=2)
    return disp, Ms


# ----------------------------------------------------------------------------- constant-space BP
def csbp_select(score, labels, k):
    """the k entries of least score, ties to the smaller label (np.lexsort), returned
    as positions into `labels`, in ascending label order"""
    order = np.lexsort((labels, score))[:k]
    return order[np.argsort(labels[order], kind="stable")]


def csbp_jacobi_step(Dc, C, IN, S, tau_q):
    """One synchronous CSBP step (R-35) in receiver storage: IN[y][x][k][i] is the
    message (x, y) receives from its neighbour in direction k, over its candidate i.
    Dc[y][x][i] = D(p, C[y][x][i]).  Message p -> q over q's candidates j:
    min_i h(i) + min(S |c_p[i] - c_q[j]|, tau_q), minus its own minimum over j."""
    H, W, k = C.shape
    OUT = np.zeros_like(IN)
    for y in range(H):
        for x in range(W):
            for kk, (dx, dy) in enumerate(DIRS):
                qx, qy = x + dx, y + dy
                if not (0 <= qx < W and 0 <= qy < H):
                    continue
                h = Dc[y, x] + sum(IN[y, x, j] for j in range(4) if j != kk)
                Vpq = np.minimum(S * np.abs(np.subtract.outer(C[y, x], C[qy, qx])), tau_q)  # [i][j]
                raw = (h[:, None] + Vpq).min(axis=0)
                OUT[qy, qx, OPP[kk]] = raw - raw.min()
    return OUT


def constant_space_bp(D0, levels, iters, k0, S, tau_q):
    """Constant-space BP (P:30 [4]; R-32..R-35) from independent pieces: numpy
    pyramid; lexsort candidate selection (top: least D; below: least D + sum of the
    parent's final incoming messages over the parent's candidates); receiver-side
    message inheritance with the edge mask; each level's checkerboard state from
    synchronous steps (the colour updated last sent Jacobi step T, the other step T-1).
    Returns (disp, candidates per level, final messages per level)."""
    Ds = [np.asarray(D0, np.int64)]
    for _ in range(levels - 1):
        Ds.append(np_pyramid(Ds[-1]))
    L = Ds[0].shape[2]
    ks = [min(L, k0 << lv) for lv in range(levels)]
    Cs, INs = [None] * levels, [None] * levels
    for lv in range(levels - 1, -1, -1):
        H, W, _ = Ds[lv].shape
        k = ks[lv]
        C = np.zeros((H, W, k), np.int64)
        IN = np.zeros((H, W, 4, k), np.int64)
        ok = neighbour_exists(H, W)
        for y in range(H):
            for x in range(W):
                if lv == levels - 1:
                    C[y, x] = csbp_select(Ds[lv][y, x], np.arange(L), k)
                else:
                    pool = Cs[lv + 1][y // 2, x // 2]
                    pin = INs[lv + 1][y // 2, x // 2]
                    sel = csbp_select(Ds[lv][y, x, pool] + pin.sum(axis=0), pool, k)
                    C[y, x] = pool[sel]
                    IN[y, x] = np.where(ok[:, y, x][:, None], pin[:, sel], 0)
        Dc = np.take_along_axis(Ds[lv], C, axis=2)
        seq = [IN]
        for _ in range(iters):
            seq.append(csbp_jacobi_step(Dc, C, seq[-1], S, tau_q))
        # the message in slot k of (x, y) was sent by the neighbour in direction k
        last = (iters - 1) % 2
        sender_last = np.zeros((H, W, 4), bool)
        for kk, (dx, dy) in enumerate(DIRS):
            sender_last[:, :, kk] = colour_mask(H, W, (last + 1) % 2)  # neighbours have the other colour
        Cs[lv], INs[lv] = C, np.where(sender_last[..., None], seq[iters], seq[iters - 1])
    bel = np.take_along_axis(Ds[0], Cs[0], axis=2) + INs[0].sum(axis=2)
    disp = np.take_along_axis(Cs[0], np.argmin(bel, axis=2)[..., None], axis=2)[..., 0]
    return disp, Cs, INs
