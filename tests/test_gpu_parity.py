"""GPU parity (-m gpu): the CUDA path through the C ABI against the CPU oracle on
the same seeded inputs.  BP (costs, every level's messages, disparities) must be
bit-exact; JBU within 1e-4 full-res px; XYZ within 1e-5 relative."""
import numpy as np
import pytest
import torch

import oracle
import synthgen

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1902_09733_b200 as P


def dev():
    return torch.device("cuda:0")


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


def run_gpu_bp(left, right, L, levels, iters, lam=0.07, dt=15.0, st=1.7, msg_bytes=0, batch=None, final=0,
               pair=2):
    """pair=2: two iterations per launch on EVERY eligible level (the default, 1,
    fuses only levels of >= 100K pixels, which small test images never reach)."""
    left = np.asarray(left)
    right = np.asarray(right)
    if left.ndim == 2:
        left, right = left[None], right[None]
    B, H, W = left.shape
    bp = P.StereoBP(W, H, L, levels, iters, lam, dt, st, batch=batch or B, msg_bytes=msg_bytes, device=dev(),
                    final=final, pair=pair)
    disp = bp.disparity(to_dev(left), to_dev(right))
    torch.cuda.synchronize()
    return bp, disp.cpu().numpy()


def check_bp_case(left, right, L, levels, iters, lam=0.07, dt=15.0, st=1.7, msg_bytes=0, all_levels=True):
    """Disparities with the fused final iteration (VSBP_OPT_FINAL) and with the
    default stored-message path, whose messages are compared on every level."""
    bp, disp = run_gpu_bp(left, right, L, levels, iters, lam, dt, st, msg_bytes)
    d_o, msgs_o = oracle.bp_disparity(left, right, L, levels, iters, lam, dt, st, return_messages=True)
    _, disp_1 = run_gpu_bp(left, right, L, levels, iters, lam, dt, st, msg_bytes, pair=0)
    assert np.array_equal(disp_1[0], d_o), "disparity differs (one iteration per launch)"
    for variant in (1, 2, 3):
        _, disp_f = run_gpu_bp(left, right, L, levels, iters, lam, dt, st, msg_bytes, final=variant)
        assert np.array_equal(disp_f[0], d_o), f"disparity differs (fused final iteration, variant {variant})"
    assert np.array_equal(disp[0], d_o), "disparity differs"
    levels_to_check = range(levels) if all_levels else [0]
    q = oracle.quantize(lam, dt, st)
    D = oracle.cost_volume(left, right, L, q)
    for l in levels_to_check:
        m_g = bp.messages(0, l).cpu().numpy()
        assert np.array_equal(m_g, msgs_o[l]), f"messages differ on level {l}"
        c_g = bp.costs(0, l).cpu().numpy()
        assert np.array_equal(c_g, D), f"costs differ on level {l}"
        if l + 1 < levels:
            D = oracle.pyramid_down(D)
    return disp[0]


# ----------------------------------------------------------------------------- BP
def test_config1_shift():
    l, r = synthgen.shifted_pair(1, 64, 48, 5)
    disp = check_bp_case(l, r, 16, 1, 5)
    assert np.mean(disp[:, 5:] == 5) >= 0.999


def test_config1_row_plane_hierarchical():
    l, r, _ = synthgen.row_plane_pair(2, 64, 48, 1, 12)
    check_bp_case(l, r, 16, 3, 5)


@pytest.mark.parametrize("seed", range(40))
def test_bp_fuzz(seed):
    rng = np.random.default_rng(1000 + seed)
    W = int(rng.choice([1, 2, 3, int(rng.integers(4, 71))]))
    H = int(rng.choice([1, 2, int(rng.integers(3, 71))]))
    L = int(rng.choice([2, 3, 16, 17, 31, 64, int(rng.integers(2, 131))]))
    levels = int(rng.integers(1, 7))
    iters = int(rng.integers(1, 13))
    lam = float(rng.choice([0.0, 0.07, 0.3, 1.0]))
    dt = float(rng.choice([1.0, 15.0, 40.0]))
    st = float(rng.choice([0.01, 1.7, 3.0, 40.0]))
    left = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    right = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    try:
        oracle.bp_disparity(left, right, L, levels, iters, lam, dt, st)
    except oracle.OracleError as e:
        with pytest.raises(P.VsbpError) as ge:
            run_gpu_bp(left, right, L, levels, iters, lam, dt, st)
        assert ge.value.code == e.code
        return
    check_bp_case(left, right, L, levels, iters, lam, dt, st)


@pytest.mark.parametrize("msg_bytes", [1, 2, 4])
def test_storage_widths_agree(msg_bytes):
    l, r, _ = synthgen.row_plane_pair(3, 97, 61, 2, 20)
    check_bp_case(l, r, 32, 4, 5, msg_bytes=msg_bytes)


def test_wide_tau_q_u16_and_i32_storage():
    rng = np.random.default_rng(5)
    l = rng.integers(0, 256, size=(33, 45), dtype=np.uint8)
    r = rng.integers(0, 256, size=(33, 45), dtype=np.uint8)
    check_bp_case(l, r, 24, 3, 4, lam=2.0, dt=60.0, st=100.0)     # tau_q = 12800 -> u16
    check_bp_case(l, r, 24, 2, 3, lam=2.0, dt=60.0, st=1000.0)    # tau_q = 128000 -> i32


@pytest.mark.parametrize("dimg", [0, 1])
@pytest.mark.parametrize("W,H,L,levels", [(13, 5, 16, 1), (64, 40, 64, 5), (33, 7, 48, 3)])
def test_level0_data_term_from_images_or_memory(W, H, L, levels, dimg):
    """VSBP_OPT_DIMG: the level-0 data term computed inside the update from the
    images (incl. the left border and the buffer's last bytes) equals reading D_0."""
    rng = np.random.default_rng(W + 3 * L + dimg)
    l = rng.integers(0, 256, size=(3, H, W), dtype=np.uint8)
    r = rng.integers(0, 256, size=(3, H, W), dtype=np.uint8)
    bp = P.StereoBP(W, H, L, levels, 5, batch=3, device=dev(), dimg=dimg)
    disp = bp.disparity(to_dev(l), to_dev(r)).cpu().numpy()
    disp_f = P.StereoBP(W, H, L, levels, 5, batch=3, device=dev(), dimg=dimg, final=2).disparity(to_dev(l), to_dev(r))
    assert np.array_equal(disp_f.cpu().numpy(), disp)
    for b in range(3):
        d_o, msgs_o = oracle.bp_disparity(l[b], r[b], L, levels, 5, return_messages=True)
        assert np.array_equal(disp[b], d_o)
        assert np.array_equal(bp.messages(b, 0).cpu().numpy(), msgs_o[0])
    D = oracle.cost_volume(l[2], r[2], L, oracle.quantize(0.07, 15.0, 1.7))
    assert np.array_equal(bp.costs(2, 0).cpu().numpy(), D)


@pytest.mark.parametrize("W,H,L,levels", [(97, 61, 32, 4), (70, 41, 130, 6), (9, 17, 64, 5)])
def test_generic_and_fused_kernels_agree_with_oracle(W, H, L, levels):
    """VSBP_OPT_KERNEL=1 (separate cost-volume, pyramid and generic update kernels)
    and the default fused/packed kernels both reproduce the oracle bit for bit."""
    rng = np.random.default_rng(W + H + L)
    l = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    r = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    d_o, msgs_o = oracle.bp_disparity(l, r, L, levels, 5, return_messages=True)
    D = oracle.cost_volume(l, r, L, oracle.quantize(0.07, 15.0, 1.7))
    assert np.array_equal(P.StereoBP(W, H, L, levels, 5, device=dev(), final=1).disparity(to_dev(l), to_dev(r))
                          .cpu().numpy(), d_o)  # fused final iteration
    for kernel in (0, 1):
        bp = P.StereoBP(W, H, L, levels, 5, kernel=kernel, device=dev())
        disp = bp.disparity(to_dev(l), to_dev(r)).cpu().numpy()
        assert np.array_equal(disp, d_o)
        Dl = D
        for lv in range(levels):
            assert np.array_equal(bp.costs(0, lv).cpu().numpy(), Dl), f"kernel {kernel} costs level {lv}"
            assert np.array_equal(bp.messages(0, lv).cpu().numpy(), msgs_o[lv])
            if lv + 1 < levels:
                Dl = oracle.pyramid_down(Dl)


@pytest.mark.parametrize("W,H,L", [(127, 19, 64), (129, 17, 49), (256, 33, 57), (301, 37, 64), (385, 18, 60)])
def test_costpyr_wide_tiles_ragged(W, H, L):
    """The 16 x 128 cost-volume tiles (levels 0-1 fused, Lp = 64): widths one
    column short of, just past and several tiles beyond 128 columns, odd heights,
    L below Lp; costs and messages on every level vs the oracle."""
    l, r, _ = synthgen.row_plane_pair(7 + W, W, H, 1, 40)
    check_bp_case(l, r, L, 4, 2)


def test_batch_equals_single():
    pairs = [synthgen.shifted_pair(10 + i, 80, 50, 3 + i) for i in range(3)]
    left = np.stack([p[0] for p in pairs])
    right = np.stack([p[1] for p in pairs])
    bp, disp = run_gpu_bp(left, right, 16, 3, 5)
    _, disp_f = run_gpu_bp(left, right, 16, 3, 5, final=2)
    assert np.array_equal(disp_f, disp)
    for i in range(3):
        assert np.array_equal(disp[i], oracle.bp_disparity(left[i], right[i], 16, 3, 5))
        _, msgs = oracle.bp_disparity(left[i], right[i], 16, 3, 5, return_messages=True)
        assert np.array_equal(bp.messages(i, 0).cpu().numpy(), msgs[0])


def test_batch_smaller_than_workspace_and_determinism():
    l, r = synthgen.shifted_pair(4, 70, 40, 6)
    bp = P.StereoBP(70, 40, 16, 2, 5, batch=4, device=dev())
    a = bp.disparity(to_dev(l), to_dev(r)).cpu().numpy()
    b = bp.disparity(to_dev(l), to_dev(r)).cpu().numpy()
    assert np.array_equal(a, b)
    assert np.array_equal(a, oracle.bp_disparity(l, r, 16, 2, 5))


def c2_pair(seed=0):
    left, right, d_lo = synthgen.stereo_pair_rgb(seed)
    return left, right, d_lo, oracle.prep(left, 4), oracle.prep(right, 4)


def test_config2_full_size_bit_exact():
    """676x380, L=64, 5 levels x 5 iterations: disparity and every level's messages."""
    _, _, d_lo, gl, gr = c2_pair(0)
    disp = check_bp_case(gl, gr, 64, 5, 5)
    assert np.mean(disp == d_lo) > 0.9


def test_config4_full_size_bit_exact():
    """1352x760, L=128, 6 levels x 8 iterations: disparity and level-0 messages."""
    left, right, d_lo = synthgen.stereo_pair_rgb(1, s=2, dmin=16, dmax=96)
    gl, gr = oracle.prep(left, 2), oracle.prep(right, 2)
    disp = check_bp_case(gl, gr, 128, 6, 8, all_levels=False)
    assert np.mean(disp == d_lo) > 0.85


# ----------------------------------------------------------------------------- a0
@pytest.mark.parametrize("s", [1, 2, 3, 4, 8])
def test_prep_bit_exact(s):
    rgb = synthgen.value_noise_rgb(20 + s, 120, 72)  # 120 x 72 divides by 1, 2, 3, 4, 8
    g = P.prep_downsample(to_dev(rgb), s).cpu().numpy()
    assert np.array_equal(g, oracle.prep(rgb, s))


@pytest.mark.parametrize("W,H,off", [(160, 76, 0), (160, 76, 4), (160, 76, 1), (64, 4, 0), (208, 36, 0)])
def test_prep_s4_kernels(W, H, off):
    """s = 4 runs a 4-pixels-per-thread kernel on 16-byte aligned rows (W % 16 == 0),
    the word kernel on 4-byte alignment and the generic one otherwise (off = byte
    offset of the frame in its buffer)."""
    frames = np.stack([synthgen.value_noise_rgb(40 + i + W, W, H) for i in range(3)])
    buf = torch.zeros(frames.size + off, dtype=torch.uint8, device=dev())
    buf[off:] = to_dev(frames.reshape(-1))
    g = P.prep_downsample(buf[off:].view(3, H, W, 3), 4).cpu().numpy()
    for i in range(3):
        assert np.array_equal(g[i], oracle.prep(frames[i], 4))


def test_prep_full_frame_batch():
    frames = np.stack([synthgen.value_noise_rgb(30 + i, 2704, 1520) for i in range(2)])
    g = P.prep_downsample(to_dev(frames), 4).cpu().numpy()
    for i in range(2):
        assert np.array_equal(g[i], oracle.prep(frames[i], 4))


# ----------------------------------------------------------------------------- a6
@pytest.mark.parametrize("s,r,ss,sr", [(2, 1, 1.3, 40.0), (3, 2, 2.0, 20.0), (4, 2, 3.75, 15.0), (4, 5, 3.75, 15.0),
                                       (2, 3, 7.5, 15.0), (1, 4, 2.0, 30.0), (5, 3, 3.0, 8.0), (8, 1, 7.5, 15.0),
                                       (6, 2, 5.0, 15.0)])
def test_jbu_small(s, r, ss, sr):
    rng = np.random.default_rng(s * 10 + r)
    lo = rng.integers(0, 64, size=(13, 19)).astype(np.int32)
    guide = synthgen.value_noise_rgb(s + r, 19 * s, 13 * s)
    got = P.jbu_upsample(to_dev(lo), to_dev(guide), s, ss, sr, r).cpu().numpy().astype(np.float64)
    ref = oracle.jbu(lo, guide, s, ss, sr, r)
    assert np.max(np.abs(got - ref)) <= 1e-4


@pytest.mark.parametrize("s,r", [(4, 6), (2, 8), (8, 7)])
def test_jbu_large_radius_scalar_path(s, r):
    """Radii above 5 (beyond the paper's 2..5) run on the one-pixel kernel: same
    tolerance vs the oracle, and still equal to the oracle near the borders."""
    rng = np.random.default_rng(100 * s + r)
    lo = rng.integers(0, 256 // s, size=(11, 17)).astype(np.int32)
    guide = synthgen.value_noise_rgb(s * r, 17 * s, 11 * s)
    got = P.jbu_upsample(to_dev(lo), to_dev(guide), s, 3.75, 15.0, r).cpu().numpy().astype(np.float64)
    ref = oracle.jbu(lo, guide, s, 3.75, 15.0, r)
    assert np.max(np.abs(got - ref)) <= 1e-4


def test_jbu_adversarial_colours():
    """Every tap far in colour from the pixel (large |logit|) still within 1e-4."""
    s, r = 4, 2
    rng = np.random.default_rng(77)
    lo = rng.integers(0, 64, size=(10, 12)).astype(np.int32)
    guide = np.where(rng.random((40, 48, 1)) < 0.5, 0, 255).astype(np.uint8).repeat(3, axis=2)
    guide = np.ascontiguousarray(guide)
    got = P.jbu_upsample(to_dev(lo), to_dev(guide), s, 3.75, 15.0, r).cpu().numpy().astype(np.float64)
    ref = oracle.jbu(lo, guide, s, 3.75, 15.0, r)
    assert np.max(np.abs(got - ref)) <= 1e-4


@pytest.mark.parametrize("s,r", [(4, 2), (2, 3), (8, 1), (4, 5)])
def test_jbu_vector_path_equals_scalar_path(s, r):
    """The P-pixels-per-thread kernel (s % P == 0, aligned buffers) and the one-pixel
    kernel (chosen when the output is misaligned) compute the same f32 arithmetic in
    the same order: bit-identical outputs."""
    rng = np.random.default_rng(5 * s + r)
    H, W = 21, 37
    lo = to_dev(rng.integers(0, 48, size=(H, W)).astype(np.int32))
    guide = to_dev(synthgen.value_noise_rgb(s * r, W * s, H * s))
    vec = P.jbu_upsample(lo, guide, s, 3.75, 15.0, r)
    buf = torch.empty(H * s * W * s + 1, dtype=torch.float32, device=dev())
    sca = P.jbu_upsample(lo, guide, s, 3.75, 15.0, r, out=buf[1:].view(1, H * s, W * s))
    assert torch.equal(vec, sca)


@pytest.mark.parametrize("s,r", [(4, 2), (2, 3), (8, 1), (4, 5)])
def test_jbu_far_pixels_vector_equals_scalar_and_oracle(s, r):
    """A guide of saturated random colours makes most pixels "far" (centre tap far in
    colour, handled warp-cooperatively by far_pixel) next to near ones in the same
    warp: both kernels bit-identical, and within 1e-4 px of the oracle."""
    rng = np.random.default_rng(11 * s + r)
    H, W = 19, 29
    # output disparities below 256 px like every BASELINE config (s*L <= 256): the
    # f32 kernel's error is relative (~2e-7), so 1e-4 px holds up to 256
    lo_np = rng.integers(0, 256 // s, size=(H, W)).astype(np.int32)
    g = np.where(rng.random((H * s, W * s, 3)) < 0.5, 0, 255).astype(np.uint8)
    g[: H * s // 2] = synthgen.value_noise_rgb(3, W * s, H * s)[: H * s // 2]  # near half
    guide = np.ascontiguousarray(g)
    lo, gd = to_dev(lo_np), to_dev(guide)
    vec = P.jbu_upsample(lo, gd, s, 3.75, 15.0, r)
    buf = torch.empty(H * s * W * s + 1, dtype=torch.float32, device=dev())
    sca = P.jbu_upsample(lo, gd, s, 3.75, 15.0, r, out=buf[1:].view(1, H * s, W * s))
    assert not torch.isnan(vec).any() and not torch.isnan(sca).any()
    bad = torch.nonzero(vec.reshape(sca.shape) != sca)
    assert bad.numel() == 0, f"vector != scalar at {bad[:8].tolist()}"
    ref = oracle.jbu(lo_np, guide, s, 3.75, 15.0, r)
    assert np.max(np.abs(vec.reshape(ref.shape).cpu().numpy().astype(np.float64) - ref)) <= 1e-4


def _jbu_tol(ref):
    """include/vsbp.h jbu_upsample_batch: 1e-4 full-res px, or one f32 ulp of the
    output where that is coarser (outputs >= 2048 px cannot be stored closer)."""
    return np.maximum(1e-4, np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64))


@pytest.mark.parametrize("s,r", [(8, 1), (8, 3), (16, 1), (16, 3), (4, 2), (2, 3)])
@pytest.mark.parametrize("labels", ["random511", "smooth_high", "steps"])
def test_jbu_whole_label_domain(s, r, labels):
    """the tolerance over the whole accepted domain -- labels up
    to 511 at s = 8 and 16 (outputs to ~8000 px).  Random labels put every window on
    the precise (double) path; a smooth high ramp keeps the fast f32 path with large
    outputs (residual accumulation); label steps mix both inside one tile.  Vector
    and scalar kernels stay bit-identical."""
    rng = np.random.default_rng(17 * s + r + len(labels))
    H, W = 15, 23
    if labels == "random511":
        lo_np = rng.integers(0, 512, size=(H, W)).astype(np.int32)
    elif labels == "smooth_high":
        lo_np = (480 + (np.arange(W)[None, :] + np.arange(H)[:, None]) // 4).astype(np.int32)
        lo_np = np.minimum(lo_np, 511)
    else:
        lo_np = np.where(np.arange(W)[None, :] < W // 2, 3, 505).repeat(H, axis=0).astype(np.int32)
        lo_np[H // 2:] += rng.integers(0, 3, size=(H - H // 2, W)).astype(np.int32)
    guide = synthgen.value_noise_rgb(s * r + 5, W * s, H * s)
    lo, gd = to_dev(lo_np), to_dev(guide)
    vec = P.jbu_upsample(lo, gd, s, 0.9 * s, 15.0, r)
    buf = torch.empty(H * s * W * s + 1, dtype=torch.float32, device=dev())
    sca = P.jbu_upsample(lo, gd, s, 0.9 * s, 15.0, r, out=buf[1:].view(1, H * s, W * s))
    assert torch.equal(vec.reshape(sca.shape), sca)
    ref = oracle.jbu(lo_np, guide, s, 0.9 * s, 15.0, r)
    got = vec.reshape(ref.shape).cpu().numpy().astype(np.float64)
    err = np.abs(got - ref)
    assert (err <= _jbu_tol(ref)).all(), (err.max(), ref.flat[np.argmax(err)])
    below = np.abs(ref) < 2048
    assert err[below].max(initial=0.0) <= 1e-4


def test_jbu_full_frame_config3():
    left, _, d_lo = synthgen.stereo_pair_rgb(2)
    got = P.jbu_upsample(to_dev(d_lo), to_dev(left), 4, 3.75, 15.0, 2).cpu().numpy().astype(np.float64)
    ref = oracle.jbu(d_lo, left, 4, 3.75, 15.0, 2)
    assert np.max(np.abs(got - ref)) <= 1e-4


# ----------------------------------------------------------------------------- a7
def test_reproject_matches_oracle():
    I = synthgen.INTRINSICS
    Q = oracle.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    assert np.array_equal(Q, P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"]))
    rng = np.random.default_rng(3)
    disp = rng.uniform(0.0, 256.0, size=(1520, 2704)).astype(np.float32)
    disp[rng.random(disp.shape) < 0.1] = 0.5  # below min_disp
    xyz_g, n_g = P.reproject(to_dev(disp), Q, 1.0)
    xyz_g = xyz_g.cpu().numpy().astype(np.float64)
    xyz_o, n_o = oracle.reproject(disp.astype(np.float64), Q, 1.0)
    assert int(n_g.cpu()[0]) == n_o
    valid = ~np.isnan(xyz_o[..., 0])
    assert np.array_equal(valid, ~np.isnan(xyz_g[..., 0]))
    err = np.linalg.norm(xyz_g[valid] - xyz_o[valid], axis=1) / np.linalg.norm(xyz_o[valid], axis=1)
    assert err.max() <= 1e-5


# ----------------------------------------------------------------------------- a0-a8
def test_pipeline_config3_end_to_end():
    left, right, _ = synthgen.stereo_pair_rgb(3)
    I = synthgen.INTRINSICS
    Q = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    pipe = P.StereoPipeline(2704, 1520, 4, 64, 5, 5, batch=2, Q=Q, device=dev())
    lt = to_dev(np.stack([left, left]))
    rt = to_dev(np.stack([right, right]))
    summ = pipe.run(lt, rt, first_pair_id=40).cpu().numpy()
    disp_o, hi_o, xyz_o, n_o = oracle.pipeline_pair(left, right, 4, 64, 5, 5, Q)
    for b in range(2):
        assert np.array_equal(pipe.disp[b].cpu().numpy(), disp_o)
        hi_g = pipe.disp_hi[b].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(hi_g - hi_o)) <= 1e-4
        ls, lh = oracle.disp_summary(disp_o)
        assert int(summ[b, 1]) == ls
        assert int(summ[b, 2]) & 0xFFFFFFFFFFFFFFFF == lh
        assert int(summ[b, 3]) == 40 + b
        # count: equal up to pixels whose disparity is within 1e-4 of min_disp
        amb = int(np.sum(np.abs(hi_o - 1.0) < 1e-4))
        assert abs(int(summ[b, 0]) - n_o) <= amb


def test_jbu_reproject_fused():
    """a6 + a7 in one kernel: disp_hi within 1e-4 px of the oracle's JBU; xyz within
    1e-5 relative of the oracle's reprojection of the SAME disp_hi; counts equal."""
    left, _, d_lo = synthgen.stereo_pair_rgb(4)
    I = synthgen.INTRINSICS
    Q = oracle.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    d_lo = d_lo.copy()
    d_lo[:40, :50] = 0  # some invalid (d < min_disp) points
    hi, xyz, n = P.jbu_reproject(to_dev(d_lo), to_dev(left), 4, 3.75, 15.0, 2, Q, 1.0)
    hi = hi[0].cpu().numpy().astype(np.float64)
    assert np.max(np.abs(hi - oracle.jbu(d_lo, left, 4, 3.75, 15.0, 2))) <= 1e-4
    xyz_o, n_o = oracle.reproject(hi, Q, 1.0)
    xyz_g = xyz[0].cpu().numpy().astype(np.float64)
    assert int(n.cpu()[0]) == n_o
    valid = ~np.isnan(xyz_o[..., 0])
    assert np.array_equal(valid, ~np.isnan(xyz_g[..., 0]))
    err = np.linalg.norm(xyz_g[valid] - xyz_o[valid], axis=1) / np.linalg.norm(xyz_o[valid], axis=1)
    assert err.max() <= 1e-5


@pytest.mark.parametrize("W,H,s,r", [(7, 5, 3, 2), (33, 9, 2, 3), (1, 1, 4, 2), (20, 3, 1, 8), (9, 9, 16, 1)])
def test_jbu_reproject_ragged(W, H, s, r):
    rng = np.random.default_rng(W * H + s)
    # f32 bound (DESIGN.md §7 a6): |err| <= s * 2^-21 * (label spread in a window);
    # keep s * spread <= 256 so 1e-4 px holds (the configurations have s <= 4)
    lo = rng.integers(0, min(40, 256 // s), size=(H, W)).astype(np.int32)
    guide = rng.integers(0, 256, size=(H * s, W * s, 3), dtype=np.uint8)
    Q = oracle.q_matrix(900.0, 880.0, W * s / 2, H * s / 2, 0.5)
    hi, xyz, n = P.jbu_reproject(to_dev(lo), to_dev(guide), s, 2.5, 20.0, r, Q, 1.0)
    hi = hi[0].cpu().numpy().astype(np.float64)
    assert np.max(np.abs(hi - oracle.jbu(lo, guide, s, 2.5, 20.0, r))) <= 1e-4
    xyz_o, n_o = oracle.reproject(hi, Q, 1.0)
    assert int(n.cpu()[0]) == n_o
    xyz_g = xyz[0].cpu().numpy().astype(np.float64)
    valid = ~np.isnan(xyz_o[..., 0])
    assert np.array_equal(valid, ~np.isnan(xyz_g[..., 0]))
    if valid.any():
        err = np.linalg.norm(xyz_g[valid] - xyz_o[valid], axis=1) / np.linalg.norm(xyz_o[valid], axis=1)
        assert err.max() <= 1e-5


# ----------------------------------------------------------------------------- f1
GOPRO_CAM = (1400.0, 1400.0, 1351.5, 759.5, -0.25, 0.08, -0.01)  # wide-angle barrel


@pytest.mark.parametrize("W,H,s,cam", [
    (64, 40, 4, (50.0, 50.0, 31.5, 19.5, 0.0, 0.0, 0.0)),
    (64, 40, 4, (40.0, 45.0, 30.0, 21.0, 0.3, 0.0, 0.0)),
    (66, 39, 3, (30.0, 30.0, 33.7, 18.2, -0.2, 0.04, 0.0)),
    (34, 18, 2, (20.0, 22.0, 16.5, 8.5, 0.1, -0.05, 0.02)),
    (23, 17, 1, (15.0, 15.0, 11.0, 8.0, -0.3, 0.1, -0.02)),
    (96, 48, 8, (60.0, 60.0, 47.5, 23.5, 0.05, 0.0, 0.01)),
    (40, 24, 4, (10.0, 10.0, 19.5, 11.5, 2.0, 0.0, 0.0)),   # strong: many sources outside the frame
])
def test_rectify_prep_bit_exact(W, H, s, cam):
    rng = np.random.default_rng(W * H + s)
    frames = [synthgen.value_noise_rgb(10 + i, W, H) for i in range(3)]
    frames[2] = rng.integers(0, 256, size=(H, W, 3), dtype=np.uint8)
    raw = to_dev(np.stack(frames))
    gray, rect = P.rectify_prep(raw, cam, s, rect=True)
    for i, f in enumerate(frames):
        rect_o, gray_o = oracle.rectify_prep(f, cam, s)
        assert np.array_equal(rect[i].cpu().numpy(), rect_o), f"rectified frame {i}"
        assert np.array_equal(gray[i].cpu().numpy(), gray_o), f"grey frame {i}"


def test_rectify_prep_full_frame_and_unaligned():
    left, right, _ = synthgen.stereo_pair_rgb(5)
    raw = to_dev(np.stack([left, right]))
    gray, rect = P.rectify_prep(raw, GOPRO_CAM, 4, rect=True)
    for i, f in enumerate([left, right]):
        rect_o, gray_o = oracle.rectify_prep(f, GOPRO_CAM, 4)
        assert np.array_equal(rect[i].cpu().numpy(), rect_o)
        assert np.array_equal(gray[i].cpu().numpy(), gray_o)
    # a frame that does not start on an 8-byte boundary takes the byte path: same result
    small = synthgen.value_noise_rgb(9, 64, 40)
    buf = torch.zeros(64 * 40 * 3 + 1, dtype=torch.uint8, device=dev())
    buf[1:] = to_dev(small).reshape(-1)
    g2, r2 = P.rectify_prep(buf[1:].view(40, 64, 3), (40.0, 45.0, 30.0, 21.0, 0.3, 0.0, 0.0), 4, rect=True)
    rect_o, gray_o = oracle.rectify_prep(small, (40.0, 45.0, 30.0, 21.0, 0.3, 0.0, 0.0), 4)
    assert np.array_equal(r2.cpu().numpy(), rect_o) and np.array_equal(g2.cpu().numpy(), gray_o)


def test_rectify_prep_rejects():
    raw = torch.zeros((1, 40, 64, 3), dtype=torch.uint8, device=dev())
    with pytest.raises(P.VsbpError) as e:
        P.rectify_prep(raw, (0.0, 50.0, 31.5, 19.5, 0, 0, 0), 4)
    assert e.value.code == -1
    with pytest.raises(P.VsbpError) as e:
        P.rectify_prep(raw, (50.0, 50.0, 31.5, 19.5, 0, 0, 0), 9)
    assert e.value.code == -1
    with pytest.raises(P.VsbpError) as e:
        P.rectify_prep(raw, (50.0, 50.0, 31.5, 19.5, 0, 0, 0), 3)
    assert e.value.code == -2
    cam = (50.0, 50.0, 31.5, 19.5, 1e12, 0, 0)
    with pytest.raises(oracle.OracleError):
        oracle.undistort_map(64, 40, cam)
    with pytest.raises(P.VsbpError) as e:
        P.rectify_prep(raw, cam, 4)
    assert e.value.code == -3


def test_pipeline_with_rectification_end_to_end():
    """f1 + a0-a8: undistorted frames through the whole path, against the oracle."""
    left, right, _ = synthgen.stereo_pair_rgb(6)
    I = synthgen.INTRINSICS
    Q = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    pipe = P.StereoPipeline(2704, 1520, 4, 64, 5, 5, batch=1, Q=Q, device=dev(), camera=GOPRO_CAM)
    summ = pipe.run(to_dev(left[None]), to_dev(right[None])).cpu().numpy()
    disp_o, hi_o, xyz_o, n_o = oracle.pipeline_pair(left, right, 4, 64, 5, 5, Q, camera=GOPRO_CAM)
    assert np.array_equal(pipe.disp[0].cpu().numpy(), disp_o)
    assert np.max(np.abs(pipe.disp_hi[0].cpu().numpy().astype(np.float64) - hi_o)) <= 1e-4
    amb = int(np.sum(np.abs(hi_o - 1.0) < 1e-4))
    assert abs(int(summ[0, 0]) - n_o) <= amb


# ----------------------------------------------------------------------------- f3
@pytest.mark.parametrize("W,H,gc,gr,K,thr", [(64, 48, 4, 3, 4, 1), (97, 61, 30, 30, 4, 10 ** 6),
                                             (33, 20, 2, 2, 16, 1), (676, 380, 30, 30, 4, 10 ** 9)])
def test_harris_corners_bit_exact(W, H, gc, gr, K, thr):
    imgs = [synthgen.value_noise_rgb(40 + i, W * 4, H * 4) for i in range(2)]
    grey = np.stack([oracle.prep(im, 4) for im in imgs])
    grey[1, 10:20, 10:30] = 128  # flat patch and ties
    R, xy, resp, cnt = P.harris_corners(to_dev(grey), gc, gr, K, thr)
    for i in range(2):
        R_o = oracle.harris_response(grey[i])
        assert np.array_equal(R[i].cpu().numpy(), R_o)
        xy_o, resp_o, cnt_o = oracle.harris_grid(R_o, gc, gr, K, thr)
        assert np.array_equal(cnt[i].cpu().numpy(), cnt_o)
        assert np.array_equal(xy[i].cpu().numpy(), xy_o)
        assert np.array_equal(resp[i].cpu().numpy(), resp_o)


def test_harris_grid_ties_on_gpu():
    """A plateau of equal responses: raster order decides, as in the oracle."""
    img = np.zeros((40, 40), np.uint8)
    for y in range(6, 34, 6):
        for x in range(6, 34, 6):
            img[y, x] = 200  # identical isolated peaks -> equal responses
    R, xy, resp, cnt = P.harris_corners(to_dev(img), 2, 2, 3, 1)
    xy_o, resp_o, cnt_o = oracle.harris_grid(oracle.harris_response(img), 2, 2, 3, 1)
    assert np.array_equal(xy.cpu().numpy(), xy_o) and np.array_equal(cnt.cpu().numpy(), cnt_o)


@pytest.mark.parametrize("r,sr", [(2, 4), (5, 16), (3, 12), (7, 20)])
def test_zssd_match_bit_exact(r, sr):
    left, right, _ = synthgen.stereo_pair_rgb(8)
    g1, g2 = oracle.prep(left, 4)[:120, :200].copy(), oracle.prep(right, 4)[:120, :200].copy()
    R = oracle.harris_response(g1)
    xy, _, _ = oracle.harris_grid(R, 6, 4, 3, 10 ** 8)
    m_g, c_g = P.zssd_match(to_dev(g1), to_dev(g2), to_dev(xy), r, sr, max_cost=2 ** 40)
    m_o, c_o = oracle.zssd_match(g1, g2, xy, r, sr, max_cost=2 ** 40)
    assert np.array_equal(m_g.cpu().numpy(), m_o)
    assert np.array_equal(c_g.cpu().numpy(), c_o)
    assert (m_o[:, 0] >= 0).sum() > 0


def test_zssd_match_constructed_shift_on_gpu():
    rng = np.random.default_rng(9)
    img = rng.integers(0, 256, size=(60, 90), dtype=np.uint8)
    sh = np.ascontiguousarray(np.roll(img, 7, axis=1))
    xy = np.array([[30, 30], [45, 20], [20, 40], [-1, -1], [2, 2]], np.int32)
    m, c = P.zssd_match(to_dev(img), to_dev(sh), to_dev(xy), 3, 8)
    m = m.cpu().numpy()
    assert np.array_equal(m[:3], xy[:3] + [7, 0]) and (m[3:] == -1).all()


def test_pipeline_features_match_oracle():
    """f3 inside the pipeline: corners of the left grey frame and their ZSSD matches
    in the right one equal the oracle's."""
    left, right, _ = synthgen.stereo_pair_rgb(10)
    I = synthgen.INTRINSICS
    Q = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    feats = dict(gc=8, gr=6, K=2, thr=10 ** 9, r=4, sr=20)
    pipe = P.StereoPipeline(2704, 1520, 4, 64, 5, 5, batch=1, Q=Q, device=dev(), features=feats)
    pipe.run(to_dev(left[None]), to_dev(right[None]))
    gl, gr = oracle.prep(left, 4), oracle.prep(right, 4)
    xy_o, _, _ = oracle.harris_grid(oracle.harris_response(gl), 8, 6, 2, 10 ** 9)
    m_o, c_o = oracle.zssd_match(gl, gr, xy_o, 4, 20)
    assert np.array_equal(pipe.corners[0].cpu().numpy(), xy_o)
    assert np.array_equal(pipe.matches[0][0].cpu().numpy(), m_o)
    assert np.array_equal(pipe.matches[1][0].cpu().numpy(), c_o)


# ----------------------------------------------------------------------------- f2
def check_csbp(left, right, L, levels, iters, k0, **kw):
    left, right = np.asarray(left), np.asarray(right)
    H, W = left.shape
    cs = P.ConstantSpaceBP(W, H, L, levels, iters, k0, batch=2, device=dev(), **kw)
    disp = cs.disparity(to_dev(np.stack([left, left])), to_dev(np.stack([right, right]))).cpu().numpy()
    d_o, cands_o = oracle.csbp_disparity(left, right, L, levels, iters, k0, return_candidates=True, **kw)
    assert np.array_equal(disp[0], d_o) and np.array_equal(disp[1], d_o)
    for lv in range(levels):
        assert np.array_equal(cs.candidates(1, lv).cpu().numpy(), cands_o[lv]), f"candidates of level {lv}"
    return disp[0]


def test_csbp_config1_shift():
    l, r = synthgen.shifted_pair(1, 64, 48, 5)
    d = check_csbp(l, r, 16, 3, 5, 2)
    assert np.mean(d[:, 5:] == 5) >= 0.999


@pytest.mark.parametrize("seed", range(16))
def test_csbp_fuzz(seed):
    rng = np.random.default_rng(2000 + seed)
    W = int(rng.choice([1, 2, 3, int(rng.integers(4, 60))]))
    H = int(rng.choice([1, 2, int(rng.integers(3, 50))]))
    L = int(rng.choice([2, 5, 16, 24, 64]))
    levels = int(rng.integers(1, 5))
    k0 = int(rng.choice([1, 2, 3, 4, 8]))
    if min(L, k0 << (levels - 1)) > 64:
        k0 = 1
    iters = int(rng.integers(1, 8))
    left = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    right = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    check_csbp(left, right, L, levels, iters, k0)


@pytest.mark.parametrize("W,H,L,levels,k0", [(37, 23, 64, 3, 16), (29, 17, 48, 2, 24), (45, 9, 64, 2, 33)])
def test_csbp_wide_candidate_sets(W, H, L, levels, k0):
    """k_l between 33 and 64 (two warps per pixel in the parallel update, C4's top
    level at k0 = 2 has k = 64)."""
    rng = np.random.default_rng(W * L + k0)
    left = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    right = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    check_csbp(left, right, L, levels, 4, k0)


def test_csbp_config2_full_size():
    """676x380, L=64, 5 levels x 5 iterations, k0=2 (k = 2,4,8,16,32)."""
    left, right, d_lo = synthgen.stereo_pair_rgb(0)
    gl, gr = oracle.prep(left, 4), oracle.prep(right, 4)
    d = check_csbp(gl, gr, 64, 5, 5, 2)
    assert np.mean(d == d_lo) > 0.8


# ----------------------------------------------------------------------------- f4
def _rot(axis, deg):
    a = np.asarray(axis, float) / np.linalg.norm(axis)
    th = np.deg2rad(deg)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K


def _icp_both(src, tgt, **kw):
    from oracle import icp
    src = np.ascontiguousarray(src, np.float32)
    tgt = np.ascontiguousarray(tgt, np.float32)
    o = icp.icp_register(src.astype(np.float64), tgt.astype(np.float64), **kw)
    g = P.icp_register(to_dev(src), to_dev(tgt), **kw).cpu().numpy()
    return o, g


@pytest.mark.parametrize("deg,shift,stride", [(5.0, 0.2, 1), (2.0, 0.5, 3), (0.0, 0.0, 1)])
def test_icp_constructed_motion_matches_oracle(deg, shift, stride):
    rng = np.random.default_rng(int(deg * 10) + stride)
    src = rng.uniform(-8, 8, size=(3000, 3)).astype(np.float32)
    src[::17] = np.nan                                   # invalid points are dropped (R-21)
    R, t = _rot([1, -2, 0.5], deg), np.array([shift, -shift / 2, shift / 3])
    tgt = (src.astype(np.float64) @ R.T + t).astype(np.float32)
    o, g = _icp_both(src, tgt, max_iter=40, max_dist=1.0, eps=1e-9, stride=stride)
    assert int(g[13]) == o["iters"] and bool(g[14]) == o["converged"]
    assert int(g[15]) == o["n_pairs"][-1]
    assert np.max(np.abs(g[:12].reshape(3, 4) - o["T"])) <= 1e-9
    assert abs(g[12] - o["rms"]) <= 1e-9


def test_icp_on_low_res_eq3_clouds():
    """Clouds of Eq.3 at BP resolution (the paper's ICP input): a pair's cloud
    against itself moved by a small rigid motion."""
    left, right, _ = synthgen.stereo_pair_rgb(3)
    gl, gr = oracle.prep(left, 4), oracle.prep(right, 4)
    d = oracle.bp_disparity(gl, gr, 64, 5, 5)
    I = synthgen.INTRINSICS
    Q = oracle.q_matrix(I["f_du"] / 4, I["f_dv"] / 4, (I["u0"] + 0.5) / 4 - 0.5, (I["v0"] + 0.5) / 4 - 0.5, I["B"])
    xyz, _ = oracle.reproject(d.astype(np.float64), Q, 1.0)
    src = xyz[120:220, 250:410].reshape(-1, 3).astype(np.float32)  # 16K points: the brute oracle stays fast
    R, t = _rot([0, 0, 1], 1.0), np.array([0.3, 0.1, -0.2])
    tgt = (src.astype(np.float64) @ R.T + t).astype(np.float32)
    o, g = _icp_both(src, tgt, max_iter=30, max_dist=2.0, eps=1e-7, stride=4)
    assert int(g[13]) == o["iters"] and int(g[15]) == o["n_pairs"][-1]
    assert np.max(np.abs(g[:12].reshape(3, 4) - o["T"])) <= 1e-8


def test_icp_failure_and_identity():
    rng = np.random.default_rng(1)
    a = rng.uniform(0, 1, size=(200, 3)).astype(np.float32)
    o, g = _icp_both(a, a + 100.0, max_iter=5, max_dist=0.5)
    assert o["iters"] == -1 and int(g[13]) == -1
    o, g = _icp_both(a, a, max_iter=5, max_dist=0.5)
    assert np.max(np.abs(g[:12].reshape(3, 4) - np.hstack([np.eye(3), np.zeros((3, 1))]))) <= 1e-12
    assert int(g[13]) == o["iters"]


# ----------------------------------------------------------------------------- bench configuration
def test_bench_launch_configuration_sampled_pairs():
    """The configuration bench.py times (C5: one batch of 256 pairs = 257 consecutive
    frames of the synthetic 2.7K video, s=4, L=64, 5x5, JBU r=2, packed clouds):
    three sampled pairs of a batch deep into the stream (first, middle, last) through
    the whole path against the oracle -- disparities bit-exact, JBU within 1e-4 px,
    the packed cloud's counts exact and its points within 1e-5 relative."""
    import bench
    from synthgen import video
    B = 256
    I = synthgen.INTRINSICS
    Q = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    pipe = P.StereoPipeline(bench.W_HI, bench.H_HI, bench.S_DOWN, bench.NDISP, bench.LEVELS, bench.ITERS, batch=B,
                            Q=Q, device=dev())
    frames = torch.empty((B + 1, bench.H_HI, bench.W_HI, 3), dtype=torch.uint8, device=dev())
    video.frames_device(bench.video_scene(1902), 17 * B, frames)
    summ = pipe.run_frames(frames, first_pair_id=17 * B).cpu().numpy()
    off = pipe.offsets.cpu().numpy()
    Qo = oracle.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    for b in (0, B // 2, B - 1):
        l, r = frames[b].cpu().numpy(), frames[b + 1].cpu().numpy()
        disp_o, hi_o, _, n_o = oracle.pipeline_pair(l, r, bench.S_DOWN, bench.NDISP, bench.LEVELS, bench.ITERS, Qo)
        assert np.array_equal(pipe.disp[b].cpu().numpy(), disp_o)
        hi_g = pipe.disp_hi[b].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(hi_g - hi_o)) <= 1e-4
        amb = int(np.sum(np.abs(hi_o - 1.0) < 1e-4))
        assert abs(int(summ[b, 0]) - n_o) <= amb and int(summ[b, 3]) == 17 * B + b
        ref = oracle.compact_cloud(hi_g, Qo, 1.0)  # the GPU's own f32 disparities: exact count
        assert off[b + 1] - off[b] == ref.shape[0] == int(summ[b, 0])
        got = pipe.xyz[off[b]:off[b + 1]].cpu().numpy().astype(np.float64)
        err = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
        assert err.max() <= 1e-5


def test_frames_run_equals_independent_pairs():
    """run_frames on n+1 consecutive frames (each frame prepped once) gives exactly
    what run() gives on the n pairs (frame j, frame j+1) passed separately."""
    from synthgen import video
    W, H, n = 512, 256, 5
    sc = video.VideoScene(77, W, H, 4, 8, 48)
    frames = torch.empty((n + 1, H, W, 3), dtype=torch.uint8, device=dev())
    video.frames_device(sc, 40, frames)
    Q = P.q_matrix(700.0, 700.0, W / 2 - 0.5, H / 2 - 0.5, 0.5)
    a = P.StereoPipeline(W, H, 4, 64, 4, 5, batch=n, Q=Q, device=dev())
    b = P.StereoPipeline(W, H, 4, 64, 4, 5, batch=n, Q=Q, device=dev())
    sa = a.run_frames(frames, first_pair_id=9)
    sb = b.run(frames[:n].contiguous(), frames[1:].contiguous(), first_pair_id=9)
    assert torch.equal(sa, sb) and torch.equal(a.disp, b.disp) and torch.equal(a.disp_hi, b.disp_hi)
    assert torch.equal(a.offsets, b.offsets)
    assert torch.equal(a.xyz[: int(a.offsets[-1])], b.xyz[: int(b.offsets[-1])])
    ld = oracle.prep(frames[2].cpu().numpy(), 4)
    assert np.array_equal(a.gray_flat[2].cpu().numpy(), ld)


def test_stream_driver_on_gpu_every_batch():
    """StereoStream end to end on the device (pinned host frame batches, copy stream,
    side-stream D2H ring smaller than the batch count): every batch's summaries reach
    on_summary in order and equal a direct run_frames of the same frames; a short
    last batch is handled."""
    from synthgen import video
    W, H, B = 256, 128, 3
    sc = video.VideoScene(5, W, H, 4, 8, 48)
    frames = torch.empty((3 * B + 1, H, W, 3), dtype=torch.uint8, device=dev())
    video.frames_device(sc, 0, frames)
    host = frames.cpu().pin_memory()
    batches = [host[0:B + 1], host[B:2 * B + 1], host[2 * B:3 * B], host[0:B + 1]]  # third is short
    Q = P.q_matrix(700.0, 700.0, W / 2 - 0.5, H / 2 - 0.5, 0.5)
    pipe = P.StereoPipeline(W, H, 4, 16, 2, 5, batch=B, Q=Q, device=dev())
    got = []
    P.StereoStream(pipe, device=dev(), ring=2).run(batches, first_pair_id=100, on_summary=lambda i, t: got.append((i, t)))
    torch.cuda.synchronize()
    assert [i for i, _ in got] == [0, 1, 2, 3]
    ref = P.StereoPipeline(W, H, 4, 16, 2, 5, batch=B, Q=Q, device=dev())
    for i, t in got:
        want = ref.run_frames(batches[i].to(dev()), first_pair_id=100 + i * B).cpu()
        assert torch.equal(t, want[: t.shape[0]]), i
    assert got[2][1].shape[0] == B - 1


def test_config4_pipeline_jbu_s2_r3():
    """C4 with its upsampling (1352x760, L=128, 6 levels x 8 iterations, JBU s=2 r=3)."""
    left, right, _ = synthgen.stereo_pair_rgb(1, s=2, dmin=16, dmax=96)
    I = synthgen.INTRINSICS
    Q = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    pipe = P.StereoPipeline(2704, 1520, 2, 128, 6, 8, batch=1, Q=Q, device=dev())
    pipe.run(to_dev(left[None]), to_dev(right[None]))
    Qo = oracle.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    disp_o, hi_o, _, _ = oracle.pipeline_pair(left, right, 2, 128, 6, 8, Qo)
    assert np.array_equal(pipe.disp[0].cpu().numpy(), disp_o)
    assert np.max(np.abs(pipe.disp_hi[0].cpu().numpy().astype(np.float64) - hi_o)) <= 1e-4


# ----------------------------------------------------------------------------- a4+a5 fused final iteration
@pytest.mark.parametrize("W,H,L,levels,iters", [(2, 1, 16, 1, 2), (3, 5, 16, 1, 3), (2, 9, 48, 2, 4), (17, 1, 32, 1, 5),
                                                (31, 23, 48, 3, 2), (64, 48, 64, 4, 5), (65, 33, 128, 5, 6),
                                                (40, 31, 64, 3, 8)])
@pytest.mark.parametrize("variant", [1, 2, 3])
def test_fused_final_iteration_matches_oracle(W, H, L, levels, iters, variant):
    """VSBP_OPT_FINAL=1: the last level-0 iteration's messages go straight
    into the receivers' beliefs.  Disparities equal the oracle and the stored-message
    path for both parities of the last colour, odd widths, 1-row images, padded label
    chunks (L = 48) and G = 8 lanes (L = 128); level-0 messages are then not exported."""
    rng = np.random.default_rng(7 * W + H + L + iters)
    l = rng.integers(0, 256, size=(2, H, W), dtype=np.uint8)
    r = np.roll(l, 3, axis=2)
    r = np.clip(r.astype(np.int32) + rng.integers(-6, 7, size=r.shape), 0, 255).astype(np.uint8)
    bp = P.StereoBP(W, H, L, levels, iters, batch=2, device=dev(), final=variant, pair=2)
    disp = bp.disparity(to_dev(l), to_dev(r)).cpu().numpy()
    ref = P.StereoBP(W, H, L, levels, iters, batch=2, device=dev(), final=0, pair=0).disparity(to_dev(l), to_dev(r))
    assert np.array_equal(disp, ref.cpu().numpy())
    for b in range(2):
        assert np.array_equal(disp[b], oracle.bp_disparity(l[b], r[b], L, levels, iters))
    with pytest.raises(RuntimeError, match="EINVAL"):
        bp.messages(0, 0)
    if levels > 1:
        bp.messages(0, 1)  # coarser levels are still materialised


# ----------------------------------------------------------------------------- a8 compaction
def _check_compaction(disp_np, Q, min_disp=1.0, batch=None):
    """compact_cloud_batch vs oracle.compact_cloud fed the same f32 disparities:
    exact counts and offsets (the validity test sees the same f32 value on both
    sides), every point within 1e-5 relative, raster order per pair."""
    B, H, W = disp_np.shape
    comp = P.CloudCompactor(W, H, batch or B, device=dev())
    xyz, off, nv = comp(to_dev(disp_np.astype(np.float32)), Q, min_disp)
    torch.cuda.synchronize()
    off = off.cpu().numpy()
    nv = nv.cpu().numpy()
    xyz = xyz.cpu().numpy().astype(np.float64)
    ref = [oracle.compact_cloud(disp_np[b].astype(np.float32).astype(np.float64), Q, min_disp) for b in range(B)]
    counts = np.array([r.shape[0] for r in ref])
    assert np.array_equal(nv, counts)
    assert np.array_equal(off, np.concatenate([[0], np.cumsum(counts)]))
    for b in range(B):
        got = xyz[off[b]:off[b + 1]]
        if counts[b]:
            err = np.linalg.norm(got - ref[b], axis=1) / np.linalg.norm(ref[b], axis=1)
            assert err.max() <= 1e-5, (b, err.max())
    return xyz, off


@pytest.mark.parametrize("B,W,H,frac", [(1, 7, 5, 0.5), (3, 45, 91, 0.7), (2, 2048, 1, 0.9), (5, 3, 700, 0.2),
                                        (4, 173, 61, 0.0), (2, 64, 64, 1.0), (9, 301, 17, 0.5)])
def test_compact_cloud_matches_oracle(B, W, H, frac):
    """Ragged segments (W not a multiple of the 128-pixel segment: a short last
    segment per row), W < 32 (lanes without pixels), exactly 16 full segments
    (W = 2048), one-row and one-column-ish shapes, empty and full pairs."""
    rng = np.random.default_rng(B * W + H)
    d = rng.uniform(1.0, 200.0, size=(B, H, W))
    d[rng.random((B, H, W)) >= frac] = rng.uniform(-5.0, 0.999)
    Q = oracle.q_matrix(900.0, 880.0, W / 2, H / 2, 0.5)
    _check_compaction(d, Q)


def test_compact_cloud_equals_dense_jbu_cloud_and_caps():
    """A packed point is bit-identical to the fused JBU+reprojection kernel's dense
    entry (same f32 Eq.3); points past cap_points are not written while offsets
    stay exact; repeated runs are deterministic."""
    s, r = 4, 2
    left, _, d_lo = synthgen.stereo_pair_rgb(4, 512, 256, s, 8, 48)
    I = synthgen.INTRINSICS
    Q = P.q_matrix(700.0, 700.0, 255.5, 127.5, I["B"])
    lo = to_dev(np.stack([d_lo, d_lo[::-1].copy()]))
    gd = to_dev(np.stack([left, left[::-1].copy()]))
    hi, dense, n = P.jbu_reproject(lo, gd, s, 3.75, 15.0, r, Q, 3.0 * s)
    comp = P.CloudCompactor(512, 256, 2, device=dev())
    xyz, off, nv = comp(hi, Q, 3.0 * s)
    torch.cuda.synchronize()
    assert torch.equal(nv, n.to(torch.int64))
    valid = ~torch.isnan(dense[..., 0])
    assert torch.equal(xyz[: int(off[-1])], dense[valid])
    xyz2, off2, _ = comp(hi, Q, 3.0 * s)
    assert torch.equal(xyz2[: int(off2[-1])], xyz[: int(off[-1])]) and torch.equal(off, off2)
    cap = int(off[1]) + 17
    small = torch.full((cap + 5, 3), 7.0, device=dev())
    xs, offs, _ = comp(hi, Q, 3.0 * s, xyz=small[:cap])
    torch.cuda.synchronize()
    assert torch.equal(offs, off)
    assert torch.equal(xs[:cap], xyz[:cap]) and bool((small[cap:] == 7.0).all())


def test_compact_cloud_full_frames_sampled():
    """BASELINE C3 size (2704 x 1520, 3 pairs, JBU output of the bench path):
    counts / offsets exact, sampled points vs the oracle."""
    left, right, d_lo = synthgen.stereo_pair_rgb(6)
    I = synthgen.INTRINSICS
    Q = P.q_matrix(I["f_du"], I["f_dv"], I["u0"], I["v0"], I["B"])
    lo = to_dev(np.stack([d_lo, d_lo, d_lo]))
    gd = to_dev(np.stack([left, left[:, ::-1].copy(), left[::-1].copy()]))
    hi = P.jbu_upsample(lo, gd, 4, 3.75, 15.0, 2)
    hi[1, :100] = 0.0  # an invalid band
    comp = P.CloudCompactor(2704, 1520, 3, device=dev())
    xyz, off, nv = comp(hi, Q, 1.0)
    torch.cuda.synchronize()
    hi_np = hi.cpu().numpy()
    counts = (hi_np >= 1.0).reshape(3, -1).sum(axis=1)
    assert np.array_equal(nv.cpu().numpy(), counts)
    assert np.array_equal(off.cpu().numpy(), np.concatenate([[0], np.cumsum(counts)]))
    rng = np.random.default_rng(0)
    xyz = xyz.cpu().numpy().astype(np.float64)
    for b in range(3):
        ref = oracle.compact_cloud(hi_np[b].astype(np.float64), Q, 1.0)
        idx = rng.integers(0, counts[b], size=2000)
        got = xyz[off.cpu().numpy()[b] + idx]
        err = np.linalg.norm(got - ref[idx], axis=1) / np.linalg.norm(ref[idx], axis=1)
        assert err.max() <= 1e-5


@pytest.mark.parametrize("s,r,W,H,B", [(4, 2, 173, 61, 3), (2, 3, 130, 47, 2), (3, 2, 41, 29, 2), (8, 1, 40, 20, 2),
                                       (4, 5, 676, 380, 1)])
def test_jbu_compact_equals_separate_calls(s, r, W, H, B):
    """jbu_compact_batch (counts folded into the JBU kernel, vector and scalar
    kernels: a 128-, 64- or 32-pixel warp row per compaction segment) ==
    jbu_upsample_batch + compact_cloud_batch, bit for bit, including pairs with
    invalid regions and rows ending in a short segment."""
    rng = np.random.default_rng(s * W + r)
    lo = rng.integers(0, 40, size=(B, H, W)).astype(np.int32)
    lo[0, : H // 3] = 0  # a band of invalid (d < min_disp) pixels
    guide = np.stack([synthgen.value_noise_rgb(b + s, W * s, H * s) for b in range(B)])
    Q = P.q_matrix(900.0, 880.0, W * s / 2, H * s / 2, 0.5)
    comp = P.CloudCompactor(W * s, H * s, B, device=dev())
    hi, xyz, off, nv = P.jbu_compact(to_dev(lo), to_dev(guide), s, 2.5, 20.0, r, Q, 1.0, comp)
    hi2 = P.jbu_upsample(to_dev(lo), to_dev(guide), s, 2.5, 20.0, r)
    xyz2, off2, nv2 = P.CloudCompactor(W * s, H * s, B, device=dev())(hi2, Q, 1.0)
    torch.cuda.synchronize()
    assert torch.equal(hi, hi2) and torch.equal(off, off2) and torch.equal(nv, nv2)
    assert torch.equal(xyz[: int(off[-1])], xyz2[: int(off2[-1])])
    assert int(off[-1]) == int((hi2 >= 1.0).sum())


@pytest.mark.gpu
def test_jbu_timing_counts_launches_and_taps():
    """jbu_timing_enable / read (bench.py's second roofline): one record per
    jbu_compact call, taps = B * sW * sH * (2r+1)^2, positive device time; nothing is
    recorded once disabled."""
    s, r, W, H, B = 4, 2, 64, 40, 2
    rng = np.random.default_rng(3)
    lo = to_dev(rng.integers(0, 20, size=(B, H, W)).astype(np.int32))
    guide = to_dev(np.stack([synthgen.value_noise_rgb(b + 1, W * s, H * s) for b in range(B)]))
    Q = P.q_matrix(900.0, 880.0, W * s / 2, H * s / 2, 0.5)
    comp = P.CloudCompactor(W * s, H * s, B, device=dev())
    P.jbu_timing_read()  # drop anything earlier
    P.jbu_timing(True)
    for _ in range(3):
        P.jbu_compact(lo, guide, s, 3.75, 15.0, r, Q, 1.0, comp)
    t = P.jbu_timing_read()
    P.jbu_timing(False)
    P.jbu_compact(lo, guide, s, 3.75, 15.0, r, Q, 1.0, comp)
    t2 = P.jbu_timing_read()
    assert t["launches"] == 3 and t["ms"] > 0
    assert t["taps"] == 3 * B * W * s * H * s * (2 * r + 1) ** 2
    assert t2["launches"] == 0 and t2["taps"] == 0
