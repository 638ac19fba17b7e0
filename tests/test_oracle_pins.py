"""Pins for the CPU oracle (-m "not gpu").  Each test checks the oracle against
something other than itself: hand-worked or SPEC-printed values (tests/golden/),
closed forms, invariants, textbook equivalences (Viterbi, Jacobi BP), exhaustive
minimisation, or a literal evaluation of the paper's equation.
lists which pin covers which oracle function."""
import math

import numpy as np
import pytest

import oracle
import synthgen
from brute import (OPP, DIRS, beliefs, brute_message, chain_min_marginals, checkerboard_via_jacobi,
                   constant_space_bp, csbp_select, energy, exhaustive_map, hierarchical_bp, jacobi_bp,
                   jbu_literal, np_cost_volume, np_pyramid, project)

Q0 = oracle.quantize(0.07, 15.0, 1.7)


# ----------------------------------------------------------------------------- O1
def test_quantize_golden(golden):
    for c in golden("quantize.json")["cases"]:
        q = oracle.quantize(c["lambda"], c["data_trunc"], c["disc_trunc"])
        assert [q.lam_q, q.tau_d, q.tau_q, q.S] == c["expect"]


@pytest.mark.parametrize("args", [(-0.1, 15, 1.7), (0.07, 0.0, 1.7), (0.07, 15, 0.0), (0.07, 0.4, 1.7),
                                  (0.07, 15, 0.003)])
def test_quantize_rejects(args):
    with pytest.raises(oracle.OracleError) as e:
        oracle.quantize(*args)
    assert e.value.code == -1


# ----------------------------------------------------------------------------- O0
def test_prep_golden(golden):
    g = golden("prep.json")
    for c in g["grey"]:
        rgb = np.array(c["rgb"], np.uint8).reshape(1, 1, 3)
        assert int(oracle.prep(rgb, 1)[0, 0]) == c["g"]
    blk = np.array(g["box2"]["grey_block"], np.uint8)
    rgb = np.repeat(blk[:, :, None], 3, axis=2)  # grey (v,v,v) -> (256v+128)>>8 = v
    assert int(oracle.prep(rgb, 2)[0, 0]) == g["box2"]["mean"]


def test_prep_mean_and_constant():
    rgb = np.full((12, 20, 3), 200, np.uint8)
    assert np.all(oracle.prep(rgb, 4) == 200)
    rgb = synthgen.value_noise_rgb(3, 64, 48)
    grey = oracle.prep(rgb, 1).astype(np.float64)
    lo = oracle.prep(rgb, 4).astype(np.float64)
    # each block mean is within 0.5 of the exact mean of the grey block (rounding)
    blocks = grey.reshape(12, 4, 16, 4).mean(axis=(1, 3))
    assert np.max(np.abs(lo - blocks)) <= 0.5 + 1e-12
    with pytest.raises(oracle.OracleError):
        oracle.prep(np.zeros((10, 10, 3), np.uint8), 3)


# ----------------------------------------------------------------------------- O2
def test_cost_volume_special_cases():
    q = oracle.QParams(lam_q=2, tau_d=15, tau_q=10, S=4)
    left = np.array([[10, 20, 200]], np.uint8)
    right = np.array([[15, 0, 190]], np.uint8)
    D = oracle.cost_volume(left, right, 3, q)
    # hand-worked: D(x,d) = 2*min(|L(x)-R(x-d)|, 15), border x-d<0 -> 2*15
    expect = np.array([[[10, 30, 30], [30, 10, 30], [20, 30, 30]]])
    assert np.array_equal(D, expect)

    img = synthgen.iid_gray(5, 40, 30)
    D = oracle.cost_volume(img, img, 16, Q0)
    assert np.all(D[:, :, 0] == 0)  # S:134 identical images
    l, r = synthgen.shifted_pair(6, 40, 30, 3)
    D = oracle.cost_volume(l, r, 16, Q0)
    assert np.all(D[:, 3:, 3] == 0)  # S:135 shifted texture
    c = np.full((8, 20), 77, np.uint8)
    D = oracle.cost_volume(c, c, 8, Q0)
    x = np.arange(20)[None, :, None]
    d = np.arange(8)[None, None, :]
    assert np.array_equal(D[0:1], np.where(x >= d, 0, Q0.lam_q * Q0.tau_d).astype(np.int32))


# ----------------------------------------------------------------------------- O3
def test_pyramid_golden(golden):
    g = golden("pyramid_3x3.json")
    Dn = oracle.pyramid_down(np.array(g["D"], np.int32))
    assert np.array_equal(Dn, np.array(g["Dn"], np.int32))


@pytest.mark.parametrize("W,H", [(1, 1), (1, 7), (7, 1), (5, 3), (8, 6), (13, 9)])
def test_pyramid_invariants(W, H):
    rng = np.random.default_rng(W * 100 + H)
    D = rng.integers(0, 1000, size=(H, W, 5)).astype(np.int32)
    Dn = oracle.pyramid_down(D)
    assert Dn.shape == ((H + 1) // 2, (W + 1) // 2, 5)
    assert np.array_equal(Dn.sum(axis=(0, 1)), D.sum(axis=(0, 1)))  # mass per label
    c = np.full((H, W, 2), 3, np.int32)
    Cn = oracle.pyramid_down(c)
    nx = np.array([min(2, W - 2 * X) for X in range((W + 1) // 2)])
    ny = np.array([min(2, H - 2 * Y) for Y in range((H + 1) // 2)])
    assert np.array_equal(Cn[:, :, 0], 3 * np.outer(ny, nx))  # children counted


# ----------------------------------------------------------------------------- O4
def test_message_golden(golden):
    for c in golden("message_hand.json")["cases"]:
        m = oracle.message(np.array(c["h"], np.int32), c["S"], c["tau_q"])
        assert m.tolist() == c["m"], c


def test_message_dt_equals_brute():
    """the O(L) two-pass DT equals the O(L^2) minimisation exactly."""
    rng = np.random.default_rng(0)
    for it in range(3000):
        L = int(rng.integers(1, 40))
        S = int(rng.choice([1, 7, 128, 256]))
        tau = int(rng.choice([1, 50, 218, 435, 5000, 1 << 20]))
        h = rng.integers(0, int(rng.choice([10, 300, 3000, 100000])), size=L).astype(np.int32)
        m = oracle.message(h, S, tau)
        assert np.array_equal(m, brute_message(h, S, tau)), (h, S, tau)
        assert m.min() == 0 and m.max() <= tau  # O5 invariants


def test_zero_cost_fixed_point():
    """all-zero costs keep all-zero messages for any number of iterations."""
    D = np.zeros((5, 7, 6), np.int32)
    M = oracle.bp_level(D, np.zeros((4, 5, 7, 6), np.int32), Q0.S, Q0.tau_q, 7)
    assert not M.any()
    img = np.full((9, 11), 50, np.uint8)
    disp, msgs = oracle.bp_disparity(img, img, 4, 3, 4, lam=0.0, return_messages=True)
    assert all(not m.any() for m in msgs)
    assert not disp.any()  # ties -> smallest d (R-13)


@pytest.mark.parametrize("seed", range(40))
def test_checkerboard_equals_jacobi(seed):
    """Bipartite grid: checkerboard BP from zero messages equals synchronous BP
    at step T on the colour updated last, and at step T-1 on the other colour."""
    rng = np.random.default_rng(seed)
    W, H, L = int(rng.integers(1, 6)), int(rng.integers(1, 5)), int(rng.integers(2, 6))
    T = int(rng.integers(1, 7))
    S, tau = int(rng.choice([1, 16, 128])), int(rng.integers(1, 400))
    D = rng.integers(0, 600, size=(H, W, L)).astype(np.int32)
    M = oracle.bp_level(D, np.zeros((4, H, W, L), np.int32), S, tau, T)
    JT = jacobi_bp(D, S, tau, T)
    JT1 = jacobi_bp(D, S, tau, T - 1)
    last = (T - 1) % 2
    for y in range(H):
        for x in range(W):
            ref = JT if (x + y) % 2 == last else JT1
            assert np.array_equal(M[:, y, x], ref[:, y, x]), (seed, x, y)


@pytest.mark.parametrize("seed", range(30))
def test_chain_beliefs_are_viterbi_min_marginals(seed):
    """H=1: tree BP is exact.  After >= 2W+2 checkerboard iterations the normalised
    Eq.1 beliefs equal the exact min-marginals, and WTA is their argmin."""
    rng = np.random.default_rng(100 + seed)
    W, L = int(rng.integers(2, 13)), int(rng.integers(2, 7))
    S, tau = int(rng.choice([16, 128])), int(rng.choice([100, 218, 400]))
    D = rng.integers(0, 700, size=(1, W, L)).astype(np.int32)
    M = oracle.bp_level(D, np.zeros((4, 1, W, L), np.int32), S, tau, 2 * W + 2)
    b = beliefs(D, M)[0]
    mu = chain_min_marginals(D[0], S, tau)
    assert np.array_equal(b - b.min(axis=1, keepdims=True), mu - mu.min(axis=1, keepdims=True))
    disp = oracle.wta(D, M)[0]
    assert np.array_equal(disp, np.argmin(mu, axis=1))
    # the WTA labelling is a global MAP of the chain (exhaustive check when tiny)
    if L ** W <= 20000:
        best, _ = exhaustive_map(D, S, tau)
        assert energy(D, disp[None, :], S, tau) == best


@pytest.mark.parametrize("seed", range(10))
def test_hierarchical_chain_forgets_init(seed):
    """levels > 1 on a 1-row image: the coarse-to-fine initialisation (pyramid +
    up-copy) is forgotten by tree BP, so enough level-0 iterations still give the
    exact min-marginals of the level-0 chain."""
    rng = np.random.default_rng(200 + seed)
    W, L = int(rng.integers(3, 14)), int(rng.integers(2, 7))
    left = rng.integers(0, 256, size=(1, W), dtype=np.uint8)
    right = rng.integers(0, 256, size=(1, W), dtype=np.uint8)
    levels = int(rng.integers(2, 4))
    disp, msgs = oracle.bp_disparity(left, right, L, levels, 2 * W + 2, return_messages=True)
    D = oracle.cost_volume(left, right, L, Q0)
    b = beliefs(D, msgs[0])[0]
    mu = chain_min_marginals(D[0], Q0.S, Q0.tau_q)
    assert np.array_equal(b - b.min(axis=1, keepdims=True), mu - mu.min(axis=1, keepdims=True))
    assert np.array_equal(disp[0], np.argmin(mu, axis=1))


HIER_PARAMS = [(0.07, 15.0, 1.7), (0.3, 40.0, 0.6), (1.0, 8.0, 3.0), (0.07, 15.0, 0.2)]


@pytest.mark.parametrize("seed", range(30))
def test_hierarchy_equals_jacobi_from_upcopy(seed):
    """P:30 [4], R-10, R-12: the whole coarse-to-fine wiring against an independent
    construction (tests/brute.py hierarchical_bp): numpy cost volume and ceil 2x2
    pyramid, np.repeat up-copy with the edge mask, and every level's checkerboard
    state rebuilt from synchronous BP started at the up-copied messages with t
    restarting at 0 on each level.  Loopy grids with few iterations do NOT forget
    their initialisation, so a wrong parent index, edge mask or colour order on any
    level changes the level-0 messages.  Every level's messages and the disparity
    must agree exactly."""
    rng = np.random.default_rng(500 + seed)
    W, H = int(rng.integers(2, 9)), int(rng.integers(2, 8))
    L = int(rng.integers(2, 6))
    levels = int(rng.integers(2, 5))
    iters = int(rng.integers(1, 7))
    lam, dt, st = HIER_PARAMS[seed % len(HIER_PARAMS)]
    left = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    right = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    q = oracle.quantize(lam, dt, st)
    disp, msgs = oracle.bp_disparity(left, right, L, levels, iters, lam, dt, st, return_messages=True)
    disp_b, msgs_b = hierarchical_bp(left, right, L, levels, iters, q)
    for lv in range(levels):
        assert np.array_equal(msgs[lv], msgs_b[lv]), (seed, lv)
    assert np.array_equal(disp, disp_b)


def _k_cheap_costs(rng, H, W, L, k, tau_q):
    """Level-0 data term where every pixel has exactly k 'cheap' labels (random
    subset, costs in [0, 600)) and the rest cost more than 600 + 4 tau_q: no
    belief of an expensive label can win, and no expensive sender label can reach
    a message's minimum (h >= min h + tau_q there)."""
    D = rng.integers(0, 600, size=(H, W, L)).astype(np.int64)
    for y in range(H):
        for x in range(W):
            exp = rng.permutation(L)[k:]
            D[y, x, exp] = 600 + 4 * tau_q + 1 + rng.integers(0, 500, size=exp.size)
    return D.astype(np.int32)


@pytest.mark.parametrize("seed", range(24))
def test_csbp_k_below_L_equals_full_bp(seed):
    """R-35 with k < L and different candidate sets at neighbouring pixels: when
    exactly k labels per pixel are cheap (the rest dominated, see _k_cheap_costs),
    one-level CSBP keeps exactly those, and its messages are the full BP's messages
    (synchronous brute BP, not the oracle) restricted to the RECEIVER's candidates
    minus their minimum; the disparities are equal.  A message that measured
    |c_p[i] - c_p[j]| instead of |c_p[i] - c_q[j]| breaks this."""
    rng = np.random.default_rng(600 + seed)
    W, H = int(rng.integers(2, 9)), int(rng.integers(1, 7))
    L = int(rng.integers(4, 11))
    k = int(rng.integers(2, L))
    iters = int(rng.integers(1, 8))
    S, tau = int(rng.choice([16, 128])), int(rng.integers(40, 420))
    D = _k_cheap_costs(rng, H, W, L, k, tau)
    disp, cands, msgs = oracle.csbp_costs(D, 1, iters, k, S, tau)
    cheap = np.sort(np.argsort(D, axis=2, kind="stable")[:, :, :k], axis=2)
    assert np.array_equal(cands[0], cheap)
    M = checkerboard_via_jacobi(D, S, tau, iters, np.zeros((4, H, W, L), np.int64))
    for y in range(H):
        for x in range(W):
            c = cands[0][y, x]
            for kk, (dx, dy) in enumerate(DIRS):
                qx, qy = x + dx, y + dy
                got = msgs[0][y, x, kk]
                if not (0 <= qx < W and 0 <= qy < H):
                    assert not got.any()
                    continue
                ref = M[OPP[kk], qy, qx][c]
                assert np.array_equal(got, ref - ref.min()), (seed, x, y, kk)
    assert np.array_equal(disp, np.argmin(beliefs(D, M), axis=2))


@pytest.mark.parametrize("seed", range(24))
def test_csbp_hierarchy_equals_brute(seed):
    """R-32..R-35 across levels against tests/brute.py constant_space_bp (numpy
    pyramid, lexsort selection by D + the parent's final incoming messages,
    receiver-side inheritance with the edge mask, synchronous O(k^2) messages with
    the truncation inside V, checkerboard state rebuilt from Jacobi steps):
    candidates, final messages and disparities of every level agree exactly."""
    rng = np.random.default_rng(700 + seed)
    W, H = int(rng.integers(2, 9)), int(rng.integers(2, 8))
    L = int(rng.integers(4, 10))
    levels = int(rng.integers(2, 4))
    k0 = int(rng.integers(1, 4))
    iters = int(rng.integers(1, 6))
    S, tau = int(rng.choice([16, 128])), int(rng.integers(40, 420))
    if seed % 2:
        D = rng.integers(0, 900, size=(H, W, L)).astype(np.int32)
    else:
        left = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
        right = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
        D = np_cost_volume(left, right, L, 9, 15).astype(np.int32)
    disp, cands, msgs = oracle.csbp_costs(D, levels, iters, k0, S, tau)
    disp_b, cands_b, msgs_b = constant_space_bp(D, levels, iters, k0, S, tau)
    for lv in range(levels):
        assert np.array_equal(cands[lv], cands_b[lv]), (seed, lv)
        assert np.array_equal(msgs[lv], msgs_b[lv]), (seed, lv)
    assert np.array_equal(disp, disp_b)


def test_csbp_selection_is_least_score_at_every_level():
    """R-34 step by step on a larger grid: level l's candidates are the k_l labels
    of the parent's pool with least D_l(p, d) + sum_k in_parent[k](d) (the parent's
    FINAL incoming messages), ties to the smaller label -- by np.lexsort."""
    rng = np.random.default_rng(11)
    H, W, L, levels, k0 = 19, 26, 20, 3, 2
    D = rng.integers(0, 2000, size=(H, W, L)).astype(np.int32)
    _, cands, msgs = oracle.csbp_costs(D, levels, 3, k0, 128, 218)
    Ds = [D.astype(np.int64)]
    for _ in range(levels - 1):
        Ds.append(np_pyramid(Ds[-1]))
    n_msg_decided = 0
    for lv in range(levels - 1):
        for y in range(Ds[lv].shape[0]):
            for x in range(Ds[lv].shape[1]):
                pool = cands[lv + 1][y // 2, x // 2]
                score = Ds[lv][y, x, pool] + msgs[lv + 1][y // 2, x // 2].sum(axis=0)
                sel = csbp_select(score, pool, cands[lv].shape[2])
                assert np.array_equal(cands[lv][y, x], pool[sel]), (lv, x, y)
                n_msg_decided += not np.array_equal(np.sort(csbp_select(Ds[lv][y, x, pool], pool, sel.size)), sel)
    assert n_msg_decided > 50  # the messages change the selection at many pixels


def test_upcopy_hand_and_constant():
    # hand-worked: parent 2x1 (L=1) right-messages [5, 0], left-messages [0, 7];
    # child 3x1: x=0,1 -> parent 0, x=2 -> parent 1; slots toward missing neighbours are 0.
    Mp = np.zeros((4, 1, 2, 1), np.int32)
    Mp[3, 0, 0, 0] = 5
    Mp[2, 0, 1, 0] = 7
    M = oracle.upcopy(Mp, 3, 1)
    assert M[3, 0, :, 0].tolist() == [5, 5, 0]
    assert M[2, 0, :, 0].tolist() == [0, 0, 7]
    assert not M[0].any() and not M[1].any()
    Mp = np.full((4, 3, 4, 2), 9, np.int32)
    M = oracle.upcopy(Mp, 7, 5)
    ok = np.ones((4, 5, 7), bool)
    ok[0, 0, :] = ok[1, 4, :] = ok[2, :, 0] = ok[3, :, 6] = False
    assert np.array_equal(M[..., 0] == 9, ok) and np.array_equal(M[..., 0] == 0, ~ok)


@pytest.mark.parametrize("seed", range(20))
def test_strong_data_is_global_map(seed):
    """If each pixel's data argmin beats every other label by > 4 tau_q, WTA equals
    the data argmin, which is then the unique global MAP (exhaustive)."""
    rng = np.random.default_rng(300 + seed)
    H, W, L = 2, 3, 3
    S, tau = 128, 218
    D = rng.integers(4 * tau + 1, 4 * tau + 400, size=(H, W, L)).astype(np.int32)
    best = rng.integers(0, L, size=(H, W))
    np.put_along_axis(D, best[..., None], 0, axis=2)
    M = oracle.bp_level(D, np.zeros((4, H, W, L), np.int32), S, tau, 5)
    disp = oracle.wta(D, M)
    assert np.array_equal(disp, best)
    e, arg = exhaustive_map(D, S, tau)
    assert len(arg) == 1 and np.array_equal(arg[0], best)


def test_loopy_energy_never_below_global_min():
    rng = np.random.default_rng(7)
    for _ in range(30):
        D = rng.integers(0, 600, size=(2, 3, 3)).astype(np.int32)
        M = oracle.bp_level(D, np.zeros((4, 2, 3, 3), np.int32), 128, 218, 5)
        disp = oracle.wta(D, M)
        best, _ = exhaustive_map(D, 128, 218)
        assert energy(D, disp, 128, 218) >= best


def test_wta_zero_messages_is_data_argmin():
    rng = np.random.default_rng(8)
    D = rng.integers(0, 1000, size=(6, 7, 9)).astype(np.int32)
    disp = oracle.wta(D, np.zeros((4, 6, 7, 9), np.int32))
    assert np.array_equal(disp, np.argmin(D, axis=2))  # argmin returns the first: ties -> smallest


def test_recovery_constant_shift_c1():
    """BASELINE config 1 (64x48, L=16, 1 level, 5 iters), shift d0=5:
    the known disparity is recovered on >= 99.9 % of pixels with x >= d0."""
    l, r = synthgen.shifted_pair(1, 64, 48, 5)
    disp = oracle.bp_disparity(l, r, 16, 1, 5)
    frac = np.mean(disp[:, 5:] == 5)
    assert frac >= 0.999, frac


def test_recovery_row_plane_hierarchical():
    """Row-wise integer plane on a 4-level pyramid: recovered away from row steps."""
    l, r, drow = synthgen.row_plane_pair(2, 160, 120, 4, 27)
    disp = oracle.bp_disparity(l, r, 32, 4, 5)
    truth = np.broadcast_to(drow[:, None], disp.shape)
    step = np.zeros(120, bool)
    step[1:] |= drow[1:] != drow[:-1]
    step[:-1] |= drow[1:] != drow[:-1]
    valid = (np.arange(160)[None, :] >= 40) & ~step[:, None]
    frac = np.mean(disp[valid] == truth[valid])
    assert frac >= 0.999, frac


def test_bp_overflow_and_args():
    img = np.zeros((4, 4), np.uint8)
    with pytest.raises(oracle.OracleError) as e:
        oracle.bp_disparity(img, img, 4, 12, 1, lam=1000.0, data_trunc=255.0)
    assert e.value.code == -3
    with pytest.raises(oracle.OracleError):
        oracle.bp_disparity(img, img, 1, 1, 1)


# ----------------------------------------------------------------------------- O7
def test_jbu_matches_literal_eq2():
    """random 4x4 low-res, random guide, vs Eq.2 evaluated literally (no
    max-subtraction), s in {2,3}."""
    rng = np.random.default_rng(9)
    for s, r in [(2, 1), (3, 2), (2, 3)]:
        lo = rng.integers(0, 30, size=(4, 4)).astype(np.int32)
        guide = rng.integers(0, 256, size=(4 * s, 4 * s, 3), dtype=np.uint8)
        got = oracle.jbu(lo, guide, s, 1.3, 40.0, r)
        ref = jbu_literal(lo, guide, s, 1.3, 40.0, r)
        assert np.max(np.abs(got - ref)) < 1e-12


def test_jbu_properties():
    rng = np.random.default_rng(10)
    s = 4
    guide = rng.integers(0, 256, size=(24, 32, 3), dtype=np.uint8)
    const = np.full((6, 8), 11, np.int32)
    assert np.allclose(oracle.jbu(const, guide, s, 3.75, 15.0, 2), s * 11, atol=1e-12, rtol=0)
    lo = rng.integers(0, 60, size=(6, 8)).astype(np.int32)
    out = oracle.jbu(lo, guide, s, 3.75, 15.0, 2)
    assert out.min() >= s * lo.min() - 1e-9 and out.max() <= s * lo.max() + 1e-9  # convex hull
    # constant guide -> spatial-only Gaussian (literal Eq.2 with g == 1)
    flat = np.full_like(guide, 90)
    assert np.max(np.abs(oracle.jbu(lo, flat, s, 3.75, 15.0, 2)
                         - jbu_literal(lo, flat, s, 3.75, 1e9, 2))) < 1e-9
    # mirror symmetry (odd s, where I_q sampling is mirror-symmetric)
    s = 3
    lo = rng.integers(0, 60, size=(5, 7)).astype(np.int32)
    guide = rng.integers(0, 256, size=(15, 21, 3), dtype=np.uint8)
    a = oracle.jbu(lo, guide, s, 2.0, 20.0, 2)
    b = oracle.jbu(lo[:, ::-1].copy(), guide[:, ::-1].copy(), s, 2.0, 20.0, 2)
    assert np.max(np.abs(a[:, ::-1] - b)) < 1e-9


def test_jbu_edge_preservation():
    """a disparity step co-located with a strong guide step (>= 5 sigma_r)
    is preserved within 5 % of the step height next to the edge."""
    s, W, H = 4, 16, 8
    lo = np.where(np.arange(W)[None, :] < 8, 10, 30).astype(np.int32).repeat(H, axis=0)
    guide = np.zeros((H * s, W * s, 3), np.uint8)
    guide[:, : 8 * s] = 40
    guide[:, 8 * s:] = 40 + 5 * 15
    out = oracle.jbu(lo, guide, s, 3.75, 15.0, 2)
    left, right = out[:, 8 * s - 1], out[:, 8 * s]
    assert np.all(np.abs(left - s * 10) <= 0.05 * s * 20)
    assert np.all(np.abs(right - s * 30) <= 0.05 * s * 20)


# ----------------------------------------------------------------------------- O8
def test_reproject_golden(golden):
    g = golden("reproject_examples.json")
    for c in g["reproject"]:
        Q = oracle.q_matrix(c["f_du"], c["f_dv"], c["u0"], c["v0"], c["B"])
        disp = np.zeros((c["v"] + 1, c["u"] + 1))
        disp[c["v"], c["u"]] = c["d"]
        xyz, n = oracle.reproject(disp, Q, 1.0)
        assert n == 1
        assert np.allclose(xyz[c["v"], c["u"]], c["xyz"], atol=1e-12)
        disp[c["v"], c["u"]] = 2 * c["d"]  # S:257 doubling d halves xyz
        xyz2, _ = oracle.reproject(disp, Q, 1.0)
        assert np.allclose(xyz2[c["v"], c["u"]], np.array(c["xyz"]) / 2, atol=1e-12)
    for c in g["project"]:
        u, v, _ = project(c["xyz"], c["f_du"], c["f_dv"], c["u0"], c["v0"], c["B"])
        assert (u, v) == tuple(c["uv"])


def test_reproject_round_trip():
    """project(first line of Eq.3) then reproject = identity to 1e-9."""
    I = synthgen.INTRINSICS
    Q = oracle.q_matrix(I["f_du"], 1390.0, I["u0"], I["v0"], I["B"])
    rng = np.random.default_rng(11)
    disp = np.zeros((40, 50))
    pts = {}
    for _ in range(200):
        u, v = int(rng.integers(0, 50)), int(rng.integers(0, 40))
        z = float(rng.uniform(5, 200))
        x = (u - I["u0"]) * z / I["f_du"]
        y = (v - I["v0"]) * z / 1390.0
        uu, vv, d = project((x, y, z), I["f_du"], 1390.0, I["u0"], I["v0"], I["B"])
        assert abs(uu - u) < 1e-9 and abs(vv - v) < 1e-9
        disp[v, u] = d
        pts[(u, v)] = (x, y, z)
    xyz, n = oracle.reproject(disp, Q, 1.0)
    for (u, v), p in pts.items():
        assert np.allclose(xyz[v, u], p, rtol=1e-9, atol=1e-9)
    assert n == int(np.sum(disp >= 1.0))
    assert np.all(np.isnan(xyz[disp < 1.0]))
    with pytest.raises(oracle.OracleError):
        oracle.reproject(disp, Q, 0.0)


# ----------------------------------------------------------------------------- a8
def test_compact_cloud_raster_order_round_trip():
    """a8 compaction (R-21): points constructed in 3-D and projected with the
    FIRST line of Eq.3 come back from the packed cloud in raster order
    (v, then u) to 1e-9; the packed list equals the dense reprojection's non-NaN
    rows; nothing valid -> no points; min_disp <= 0 rejected."""
    I = synthgen.INTRINSICS
    Q = oracle.q_matrix(I["f_du"], 1390.0, I["u0"], I["v0"], I["B"])
    rng = np.random.default_rng(12)
    H, W = 31, 47
    disp = np.where(rng.random((H, W)) < 0.3, 0.5, 0.0)  # invalid background (d < 1)
    pts = {}
    for _ in range(300):
        u, v = int(rng.integers(0, W)), int(rng.integers(0, H))
        z = float(rng.uniform(5, 200))
        x = (u - I["u0"]) * z / I["f_du"]
        y = (v - I["v0"]) * z / 1390.0
        disp[v, u] = project((x, y, z), I["f_du"], 1390.0, I["u0"], I["v0"], I["B"])[2]
        pts[(v, u)] = (x, y, z)
    got = oracle.compact_cloud(disp, Q, 1.0)
    want = np.array([pts[k] for k in sorted(pts)])
    assert got.shape == want.shape
    assert np.allclose(got, want, rtol=1e-9, atol=1e-9)
    dense, n = oracle.reproject(disp, Q, 1.0)
    assert n == got.shape[0]
    assert np.array_equal(got, dense[~np.isnan(dense[..., 0])])
    assert oracle.compact_cloud(np.zeros((4, 5)), Q, 1.0).shape == (0, 3)
    with pytest.raises(oracle.OracleError):
        oracle.compact_cloud(disp, Q, 0.0)


def test_disp_summary_hash_known_value():
    # SplitMix64 seeded with 0 yields 0xE220A8397B1DCDAF as its first output,
    # which is mix(0) here: one pixel at index 0 with label 0.
    s, h = oracle.disp_summary(np.zeros((1, 1), np.int32))
    assert s == 0 and h == 0xE220A8397B1DCDAF
    d = np.array([[3, 4]], np.int32)
    s, _ = oracle.disp_summary(d)
    assert s == 7


# ----------------------------------------------------------------------------- f1 rectification
def test_undistort_map_golden(golden):
    """Hand-worked radial maps (P:26 radial only; R-26)."""
    for case in golden("undistort.json")["cases"]:
        u, v = case["uv"]
        mx, my = oracle.undistort_map(u + 3, v + 3, case["cam"])
        assert [int(mx[v, u]), int(my[v, u])] == case["map"], case["note"]


def test_undistort_zero_distortion_is_identity_and_principal_point_fixed():
    mx, my = oracle.undistort_map(37, 23, (31.0, 29.0, 17.3, 9.6, 0.0, 0.0, 0.0))
    vv, uu = np.mgrid[0:23, 0:37]
    assert np.array_equal(mx, 32 * uu) and np.array_equal(my, 32 * vv)  # S:67 identity
    for k in [(0.3, 0, 0), (-0.2, 0.05, 0.01), (0, 0, 1.0)]:
        mx, my = oracle.undistort_map(41, 31, (40.0, 40.0, 20.0, 15.0) + k)
        assert mx[15, 20] == 32 * 20 and my[15, 20] == 32 * 15  # principal point


def test_undistort_radial_symmetry():
    """Radial model: mirror-symmetric about the principal point, the displacement
    is along the ray from it, and |src - c| grows with k1 > 0 (barrel correction)."""
    W = H = 41
    mx, my = oracle.undistort_map(W, H, (30.0, 30.0, 20.0, 20.0, 0.2, 0.0, 0.0))
    assert np.array_equal(mx - 640, -(mx[:, ::-1] - 640))
    assert np.array_equal(my - 640, -(my[::-1, :] - 640))
    vv, uu = np.mgrid[0:H, 0:W]
    du, dv = uu - 20, vv - 20
    r_dst = np.hypot(du, dv)
    r_src = np.hypot(mx / 32 - 20, my / 32 - 20)
    assert np.all(r_src >= r_dst - 1 / 32)
    cross = (mx / 32 - 20) * dv - (my / 32 - 20) * du
    assert np.max(np.abs(cross)) <= r_dst.max() / 32 + 1e-9


def test_remap_identity_shift_and_ramp():
    rng = np.random.default_rng(11)
    img = rng.integers(0, 256, size=(9, 13, 3), dtype=np.uint8)
    vv, uu = np.mgrid[0:9, 0:13].astype(np.int32)
    assert np.array_equal(oracle.remap_rgb(img, 32 * uu, 32 * vv), img)  # S:72 identity
    sh = oracle.remap_rgb(img, 32 * (uu + 1), 32 * vv)                     # S:73 integer shift
    assert np.array_equal(sh[:, :-1], img[:, 1:]) and not sh[:, -1].any()
    ramp = np.broadcast_to((2 * np.arange(13, dtype=np.uint8))[None, :, None], (9, 13, 3)).copy()
    half = oracle.remap_rgb(ramp, 32 * uu + 16, 32 * vv)                   # S:74 half-pixel ramp
    assert np.array_equal(half[:, :-1, 0], (2 * uu + 1)[:, :-1])
    assert np.array_equal(half[:, -1, 0], (ramp[:, -1, 0].astype(int) + 1) // 2)  # right tap is outside (0)


def test_remap_is_exact_on_affine_images():
    """Bilinear interpolation reproduces an affine image exactly, so with the
    integer weights the output is the affine value at the 1/32-px source point
    rounded half up (R-27)."""
    rng = np.random.default_rng(12)
    H, W = 20, 30
    a, b, c = 3, 5, 7  # I = 3u + 5v + 7 <= 3*29 + 5*19 + 7 = 189
    vv, uu = np.mgrid[0:H, 0:W]
    img = np.repeat((a * uu + b * vv + c).astype(np.uint8)[..., None], 3, axis=2)
    mx = rng.integers(0, 32 * (W - 1), size=(H, W)).astype(np.int32)
    my = rng.integers(0, 32 * (H - 1), size=(H, W)).astype(np.int32)
    out = oracle.remap_rgb(img, mx, my)[..., 1].astype(np.int64)
    num = a * mx.astype(np.int64) + b * my.astype(np.int64) + 32 * c   # 32 * exact value
    assert np.array_equal(out, (num + 16) // 32)


def test_rectify_prep_without_distortion_is_prep():
    rgb = synthgen.value_noise_rgb(3, 64, 40)
    rect, grey = oracle.rectify_prep(rgb, (50.0, 50.0, 31.5, 19.5, 0.0, 0.0, 0.0), 4)
    assert np.array_equal(rect, rgb)
    assert np.array_equal(grey, oracle.prep(rgb, 4))


def test_undistort_domain_rejects_runaway_maps():
    """R-26 domain: a map whose bound leaves |coordinate| < 2^24 px is rejected."""
    with pytest.raises(oracle.OracleError) as e:
        oracle.undistort_map(64, 40, (50.0, 50.0, 31.5, 19.5, 1e12, 0.0, 0.0))
    assert e.value.code == -3
    with pytest.raises(oracle.OracleError):
        oracle.undistort_map(64, 40, (0.0, 50.0, 31.5, 19.5, 0.0, 0.0, 0.0))


# ----------------------------------------------------------------------------- f3 Harris + ZSSD
I64_MIN = np.iinfo(np.int64).min


def test_harris_closed_forms():
    """R-28 pinned by closed forms of the binomial-window Harris response
    (Eq.4-5): sum b = 16, sum b i^2 = 16 for b = {1,4,6,4,1}."""
    H = W = 16
    vv, uu = np.mgrid[0:H, 0:W]
    R = oracle.harris_response(np.zeros((H, W), np.uint8))
    assert (R[3:H - 3, 3:W - 3] == 0).all() and (R[:3] == I64_MIN).all() and (R[:, -3:] == I64_MIN).all()
    # linear ramp I = 3x + 5y: A = 6, B = 10 everywhere -> det = 0, R25 = -(256 (36 + 100))^2
    R = oracle.harris_response((3 * uu + 5 * vv).astype(np.uint8))
    assert (R[3:H - 3, 3:W - 3] == -(256 * 136) ** 2).all()
    # saddle I = x y: Sxx = 1024 (y^2+1), Syy = 1024 (x^2+1), Sxy = 1024 x y
    R = oracle.harris_response((uu * vv).astype(np.uint8))
    x, y = uu[3:H - 3, 3:W - 3].astype(np.int64), vv[3:H - 3, 3:W - 3].astype(np.int64)
    expect = 25 * 1024 ** 2 * (x * x + y * y + 1) - 1024 ** 2 * (x * x + y * y + 2) ** 2
    assert np.array_equal(R[3:H - 3, 3:W - 3], expect)


def test_harris_rotation_invariance_and_edges():
    rng = np.random.default_rng(21)
    img = rng.integers(0, 256, size=(23, 23), dtype=np.uint8)
    R = oracle.harris_response(img)
    Rr = oracle.harris_response(np.ascontiguousarray(np.rot90(img)))
    assert np.array_equal(np.rot90(R), Rr)                     # "invariant to rotation"
    step = np.zeros((20, 20), np.uint8)
    step[:, 10:] = 200
    assert (oracle.harris_response(step)[3:-3, 3:-3] <= 0).all()  # straight edge: R <= 0
    quad = np.zeros((20, 20), np.uint8)
    quad[10:, 10:] = 200
    Rq = oracle.harris_response(quad)
    iy, ix = np.unravel_index(np.argmax(np.where(Rq == I64_MIN, I64_MIN, Rq)), Rq.shape)
    assert Rq[iy, ix] > 0 and abs(iy - 9.5) <= 1.5 and abs(ix - 9.5) <= 1.5  # a corner responds at the corner


def test_harris_single_pixel():
    img = np.zeros((41, 41), np.uint8)
    img[20, 20] = 255
    xy, resp, cnt = oracle.harris_grid(oracle.harris_response(img), 1, 1, 4, 1)
    assert cnt[0] >= 1 and abs(xy[0, 0] - 20) <= 1 and abs(xy[0, 1] - 20) <= 1


def _brute_grid(R, gc, gr, K, thr):
    H, W = R.shape
    out = []
    for j in range(gr):
        for i in range(gc):
            x0, x1 = i * W // gc, (i + 1) * W // gc
            y0, y1 = j * H // gr, (j + 1) * H // gr
            cand = []
            for y in range(max(y0, 4), min(y1, H - 4)):
                for x in range(max(x0, 4), min(x1, W - 4)):
                    r = R[y, x]
                    nb = R[y - 1:y + 2, x - 1:x + 2].copy()
                    nb[1, 1] = I64_MIN
                    if r >= thr and (nb < r).all():
                        cand.append((-int(r), y, x))
            cand.sort()
            out.append([(x, y, -r) for r, y, x in cand[:K]])
    return out


@pytest.mark.parametrize("seed", range(6))
def test_harris_grid_matches_brute_selection(seed):
    """R-29: per-cell top-K strict maxima, ties to raster order -- against a sort."""
    rng = np.random.default_rng(seed)
    H, W = int(rng.integers(12, 40)), int(rng.integers(12, 40))
    R = rng.integers(0, 6, size=(H, W)).astype(np.int64) * 10  # many ties
    gc, gr, K = int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 4))
    xy, resp, cnt = oracle.harris_grid(R, gc, gr, K, 10)
    for c, want in enumerate(_brute_grid(R, gc, gr, K, 10)):
        assert cnt[c] == len(want)
        for k, (x, y, r) in enumerate(want):
            assert (xy[c * K + k, 0], xy[c * K + k, 1], resp[c * K + k]) == (x, y, r)
        assert (xy[c * K + len(want):(c + 1) * K] == -1).all()


def test_zssd_definition_and_properties():
    from fractions import Fraction
    rng = np.random.default_rng(3)
    a = rng.integers(0, 256, size=(15, 15), dtype=np.uint8)
    b = rng.integers(0, 256, size=(15, 15), dtype=np.uint8)
    r = 2
    n = (2 * r + 1) ** 2
    pa = a[5:10, 6:11].astype(int)
    pb = b[4:9, 7:12].astype(int)
    ma, mb = Fraction(int(pa.sum()), n), Fraction(int(pb.sum()), n)
    z = sum(((Fraction(int(u)) - ma) - (Fraction(int(v)) - mb)) ** 2 for u, v in zip(pa.ravel(), pb.ravel()))
    assert oracle.zssd(a, b, 8, 7, 9, 6, r) == n * z                          # S:320 definition
    assert oracle.zssd(a, a, 8, 7, 8, 7, r) == 0                               # identical patches
    c = np.clip(a.astype(int) + 17, 0, 255).astype(np.uint8)
    a2 = np.clip(a, 0, 238).astype(np.uint8)
    assert oracle.zssd(a2, (a2 + 17).astype(np.uint8), 8, 7, 8, 7, r) == 0     # bias invariance
    assert oracle.zssd(a, b, 8, 7, 9, 6, r) == oracle.zssd(b, a, 9, 6, 8, 7, r)  # symmetry
    with pytest.raises(oracle.OracleError):
        oracle.zssd(a, b, 1, 7, 9, 6, r)
    del c


def test_zssd_match_self_shift_and_textureless():
    rng = np.random.default_rng(4)
    img = rng.integers(0, 256, size=(40, 60), dtype=np.uint8)
    xy = np.array([[20, 20], [30, 15], [12, 25], [-1, -1]], np.int32)
    m, c = oracle.zssd_match(img, img, xy, 3, 8)
    assert np.array_equal(m[:3], xy[:3]) and (c[:3] == 0).all() and (m[3] == -1).all()  # S:330 self-match
    sh = np.roll(img, 7, axis=1)                                                  # img2(x+7) = img1(x)
    m, c = oracle.zssd_match(img, sh, xy, 3, 8)
    assert np.array_equal(m[:3], xy[:3] + [7, 0]) and (c[:3] == 0).all()        # S:331 shift by (7,0)
    flat = np.full_like(img, 90)
    m, c = oracle.zssd_match(img, flat, xy, 3, 8)
    assert (m == -1).all()                                                         # S:332 ambiguity rejected
    m, c = oracle.zssd_match(img, sh, xy, 3, 8, max_cost=0)
    assert np.array_equal(m[:3], xy[:3] + [7, 0])


# ----------------------------------------------------------------------------- f2 constant-space BP
@pytest.mark.parametrize("seed", range(12))
def test_csbp_single_level_all_labels_is_bp(seed):
    """R-32..R-35 with one level and k >= L: every label is a candidate, messages are
    the O(k^2) minimisation -- the full BP of O4 (Eq.1), label for label."""
    rng = np.random.default_rng(300 + seed)
    W, H, L = int(rng.integers(1, 14)), int(rng.integers(1, 10)), int(rng.integers(2, 12))
    l = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    r = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    it = int(rng.integers(1, 8))
    assert np.array_equal(oracle.csbp_disparity(l, r, L, 1, it, L + int(rng.integers(0, 3))),
                          oracle.bp_disparity(l, r, L, 1, it))


@pytest.mark.parametrize("seed", range(10))
def test_csbp_chain_reaches_a_map_labelling(seed):
    """On a chain (tree) BP converges to the exact min-marginals whatever the
    coarse-level initialisation, so with all labels kept the WTA labelling has the
    exhaustive minimum energy (unique-MAP draws)."""
    rng = np.random.default_rng(400 + seed)
    W, L = int(rng.integers(3, 8)), 3
    l = rng.integers(0, 256, size=(1, W), dtype=np.uint8)
    r = rng.integers(0, 256, size=(1, W), dtype=np.uint8)
    q = oracle.quantize(0.07, 15.0, 1.7)
    D = oracle.cost_volume(l, r, L, q)
    best, _ = exhaustive_map(D, q.S, q.tau_q)
    f = oracle.csbp_disparity(l, r, L, 3, 2 * W + 4, L)
    assert energy(D, f, q.S, q.tau_q) == best


def test_csbp_candidates_selection_and_nesting():
    rng = np.random.default_rng(7)
    H, W, L, levels, k0 = 21, 30, 24, 3, 3
    l = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    r = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    _, cands = oracle.csbp_disparity(l, r, L, levels, 4, k0, return_candidates=True)
    ks = oracle.csbp_k(L, levels, k0)
    assert [c.shape[2] for c in cands] == ks == [3, 6, 12]
    q = oracle.quantize(0.07, 15.0, 1.7)
    D = oracle.cost_volume(l, r, L, q)
    for _ in range(levels - 1):
        D = oracle.pyramid_down(D)
    # top level: the k least data costs, ties to the smaller label (stable sort)
    top = np.sort(np.argsort(D, axis=2, kind="stable")[:, :, :ks[-1]], axis=2)
    assert np.array_equal(cands[-1], top)
    for lv in range(levels - 1):
        c, cp = cands[lv], cands[lv + 1]
        assert (np.diff(c, axis=2) > 0).all()  # ascending, distinct
        for y in range(c.shape[0]):
            for x in range(c.shape[1]):
                assert set(c[y, x]) <= set(cp[y // 2, x // 2])  # nested in the parent's (R-34)


def test_csbp_recovers_constant_and_row_plane_shift():
    l, r = synthgen.shifted_pair(1, 64, 48, 5)
    d = oracle.csbp_disparity(l, r, 16, 3, 5, 2)
    assert np.mean(d[:, 5:] == 5) >= 0.999
    l, r, drow = synthgen.row_plane_pair(2, 160, 120, 4, 27)
    disp = oracle.csbp_disparity(l, r, 32, 4, 5, 2)
    truth = np.broadcast_to(drow[:, None], disp.shape)
    step = np.zeros(120, bool)
    step[1:] |= drow[1:] != drow[:-1]
    step[:-1] |= drow[1:] != drow[:-1]
    valid = (np.arange(160)[None, :] >= 40) & ~step[:, None]
    frac = np.mean(disp[valid] == truth[valid])
    assert frac >= 0.99, frac


# ----------------------------------------------------------------------------- f4 ICP
def _rot(axis, deg):
    a = np.asarray(axis, float) / np.linalg.norm(axis)
    th = np.deg2rad(deg)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K  # Rodrigues


def test_icp_identity_and_constructed_motion():
    from oracle import icp
    rng = np.random.default_rng(5)
    src = rng.uniform(-5, 5, size=(400, 3))
    r = icp.icp_register(src, src, max_iter=5)
    assert np.allclose(r["T"], np.hstack([np.eye(3), np.zeros((3, 1))]), atol=1e-12) and r["rms"] <= 1e-12
    R, t = _rot([1, 2, 3], 5.0), np.array([0.2, -0.1, 0.15])
    tgt = src @ R.T + t                                                   # 5 deg, 0.2 m
    r = icp.icp_register(src, tgt, max_iter=60, max_dist=2.0, eps=1e-12)
    assert np.allclose(r["T"][:, :3], R, atol=1e-6) and np.allclose(r["T"][:, 3], t, atol=1e-6)
    assert all(b <= a + 1e-12 for a, b in zip(r["rms_history"], r["rms_history"][1:]))  # S:480 monotone


def test_icp_rigid_update_is_the_least_squares_motion():
    """Exact correspondences: the SVD update recovers the motion in one step and is
    a proper rotation (det +1) -- also for a mirrored-looking planar set."""
    from oracle import icp
    rng = np.random.default_rng(6)
    p = rng.normal(size=(50, 3))
    R, t = _rot([0, 0, 1], 40.0), np.array([1.0, 2.0, 3.0])
    T = icp.rigid_update(p, p @ R.T + t)
    assert np.allclose(T[:, :3], R, atol=1e-12) and np.allclose(T[:, 3], t, atol=1e-12)
    flat = p.copy()
    flat[:, 2] = 0.0
    T = icp.rigid_update(flat, flat @ R.T + t)
    assert abs(np.linalg.det(T[:, :3]) - 1.0) < 1e-12


def test_icp_far_clouds_fail_and_nan_rows_dropped():
    from oracle import icp
    rng = np.random.default_rng(7)
    a = rng.uniform(0, 1, size=(100, 3))
    r = icp.icp_register(a, a + 100.0, max_dist=0.5)
    assert r["iters"] == -1                                                # S:476 no pairs
    b = a.copy()
    b[::3] = np.nan
    r1 = icp.icp_register(b, a, max_iter=3)
    assert r1["n_pairs"][0] == np.sum(~np.isnan(b[:, 0]))


def test_icp_nearest_is_brute_force_minimum():
    from oracle import icp
    rng = np.random.default_rng(8)
    P, Q = rng.normal(size=(37, 3)), rng.normal(size=(53, 3))
    j, d2 = icp.nearest(P, Q, chunk=5)
    full = ((P[:, None, :] - Q[None, :, :]) ** 2).sum(axis=2)
    assert np.array_equal(j, full.argmin(axis=1)) and np.allclose(d2, full.min(axis=1), rtol=1e-15)


# ----------------------------------------------------------------------------- the pins bite
def test_oracle_mutations_are_caught():
    """tools/mutation_check.py: every plausible mistake listed there (t carried
    across levels, wrong parent index, cp[j] for cq[j], pool scored by D only, ...)
    makes at least one pin above fail; documented equivalent mutants excepted."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "mutation_check.py"), "--fast"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
