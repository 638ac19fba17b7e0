"""Guard-band checks of every kernel family (-m gpu) -- the substitute for
compute-sanitizer, which this GPU pool refuses to run (profiles/r02_sanitizer_unavailable.txt).

Every device buffer a call touches (inputs, outputs, workspaces) is a view into a
larger allocation with PAD bytes on both sides:
  * out-of-bounds WRITES: the pads of every buffer must come back untouched;
  * out-of-bounds READS that matter: each call runs twice, with the input pads
    filled with 0x00 and with 0xFF, and the outputs must be bitwise identical;
  * uninitialised reads of outputs / workspaces: those buffers are pre-filled with
    a different pattern in each run (0x00 / 0xFF) -- identical results mean no
    kernel reads an output or scratch byte before writing it;
  * races: the two runs must also agree with a third plain run (bitwise).
The shapes are small and ragged (tails in every tiled dimension)."""
import ctypes as C

import numpy as np
import pytest
import torch

import synthgen

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1902_09733_b200 as P

PAD = 4096


class Arena:
    """Device buffers with guard pads; fill(pattern) resets pads (and, for outputs,
    the payload) before a run."""

    def __init__(self):
        self.bufs = []

    def add(self, nbytes: int, payload: np.ndarray | None = None, kind: str = "in"):
        nb = ((nbytes + 255) // 256) * 256
        raw = torch.empty(nb + 2 * PAD, dtype=torch.uint8, device="cuda")
        self.bufs.append((raw, nbytes, payload, kind))
        return raw[PAD:PAD + nbytes]

    def fill(self, pat: int):
        for raw, n, payload, kind in self.bufs:
            raw.fill_(pat)
            if payload is not None:
                raw[PAD:PAD + n].copy_(torch.from_numpy(np.ascontiguousarray(payload).view(np.uint8).reshape(-1)))

    def pads_intact(self, pat: int):
        for raw, n, _, _ in self.bufs:
            if not bool((raw[:PAD] == pat).all()) or not bool((raw[PAD + n:] == pat).all()):
                return False
        return True

    def outputs(self):
        return [raw[PAD:PAD + n].clone() for raw, n, _, kind in self.bufs if kind == "out"]


def t(buf: torch.Tensor, dtype, shape):
    return buf.view(dtype).view(shape)


def run_guarded(setup, call, post=None):
    """setup(arena) -> state; call(state) enqueues the op; post(state) -> extra
    tensors to compare (e.g. the written prefix of a packed output).  Runs with pads
    0x00 and 0xFF, then a third time; asserts pads intact and outputs identical."""
    results = []
    for pat in (0x00, 0xFF, 0x00):
        ar = Arena()
        st = setup(ar)
        ar.fill(pat)
        call(st)
        torch.cuda.synchronize()
        assert ar.pads_intact(pat), "a kernel wrote outside its buffers"
        results.append(ar.outputs() + ([x.clone() for x in post(st)] if post else []))
    for a, b in zip(results[0], results[1]):
        assert torch.equal(a, b), "output depends on bytes outside the inputs or on stale output/scratch bytes"
    for a, b in zip(results[0], results[2]):
        assert torch.equal(a, b), "non-deterministic output"


def _ptr(x):
    return C.c_void_p(x.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


# ----------------------------------------------------------------------------- a0 / f1
@pytest.mark.parametrize("W,H,s", [(2704, 16, 4), (100, 36, 4), (64, 24, 8), (33, 21, 3)])
def test_guard_prep(W, H, s):
    rng = np.random.default_rng(W + H)
    n = 3
    rgb = rng.integers(0, 256, size=(n, H, W, 3), dtype=np.uint8)

    def setup(ar):
        return ar.add(rgb.nbytes, rgb), ar.add(n * (H // s) * (W // s), kind="out")

    def call(st):
        i, o = st
        assert P.lib().prep_downsample_batch(n, _ptr(i), W, H, s, _ptr(o), _stream()) == 0

    run_guarded(setup, call)


def test_guard_rectify():
    W, H, s, n = 128, 64, 4, 2
    rgb = np.random.default_rng(1).integers(0, 256, size=(n, H, W, 3), dtype=np.uint8)
    cam = (C.c_double * 7)(70.0, 70.0, 63.5, 31.5, -0.25, 0.08, -0.01)

    def setup(ar):
        return ar.add(rgb.nbytes, rgb), ar.add(n * (H // s) * (W // s), kind="out"), ar.add(rgb.nbytes, kind="out")

    def call(st):
        i, g, r = st
        assert P.lib().rectify_prep_batch(n, _ptr(i), W, H, cam, s, _ptr(g), _ptr(r), _stream()) == 0

    run_guarded(setup, call)


# ----------------------------------------------------------------------------- a1-a5
@pytest.mark.parametrize("W,H,L,levels,iters,msg_bytes,kernel,final,pair", [
    (45, 31, 64, 4, 5, 0, 0, 0, 1), (45, 31, 64, 4, 5, 0, 0, 2, 1), (37, 19, 48, 3, 4, 0, 0, 1, 1),
    (33, 17, 24, 3, 3, 2, 0, 0, 1), (29, 13, 16, 2, 5, 4, 1, 0, 1), (70, 9, 128, 5, 6, 0, 0, 0, 1),
    (45, 31, 64, 4, 5, 0, 0, 0, 2), (133, 70, 64, 3, 7, 0, 0, 0, 2), (70, 9, 128, 5, 6, 0, 0, 0, 2),
    (37, 19, 48, 3, 4, 0, 0, 0, 2), (133, 70, 64, 3, 5, 0, 0, 3, 2), (37, 19, 48, 3, 4, 0, 0, 3, 2)])
def test_guard_bp(W, H, L, levels, iters, msg_bytes, kernel, final, pair):
    """pair = 2: two iterations per launch on every level (cp.async staging, the
    shared-memory ring, the second message array)."""
    rng = np.random.default_rng(W * L + final)
    B = 2
    left = rng.integers(0, 256, size=(B, H, W), dtype=np.uint8)
    right = rng.integers(0, 256, size=(B, H, W), dtype=np.uint8)
    bp = P.StereoBP(W, H, L, levels, iters, batch=B, msg_bytes=msg_bytes, kernel=kernel, final=final, device="cuda",
                    pair=pair)
    nbytes = bp.workspace.numel()

    def setup(ar):
        return ar.add(left.nbytes, left), ar.add(right.nbytes, right), ar.add(B * H * W * 4, kind="out"), \
            ar.add(nbytes, kind="scratch")

    def call(st):
        l, r, d, ws = st
        assert P.lib().bp_set_workspace(bp._h, _ptr(ws), nbytes, B) == 0
        assert P.lib().bp_disparity_batch(bp._h, B, _ptr(l), _ptr(r), _ptr(d), _stream()) == 0

    run_guarded(setup, call)


def test_guard_csbp():
    W, H, L, levels, iters, k0, B = 41, 23, 32, 3, 4, 2, 2
    rng = np.random.default_rng(5)
    left = rng.integers(0, 256, size=(B, H, W), dtype=np.uint8)
    right = rng.integers(0, 256, size=(B, H, W), dtype=np.uint8)
    cs = P.ConstantSpaceBP(W, H, L, levels, iters, k0, batch=B, device="cuda")
    nbytes = cs.workspace.numel()

    def setup(ar):
        return ar.add(left.nbytes, left), ar.add(right.nbytes, right), ar.add(B * H * W * 4, kind="out"), \
            ar.add(nbytes, kind="scratch")

    def call(st):
        l, r, d, ws = st
        assert P.lib().csbp_set_workspace(cs._h, _ptr(ws), nbytes, B) == 0
        assert P.lib().csbp_disparity_batch(cs._h, B, _ptr(l), _ptr(r), _ptr(d), _stream()) == 0

    run_guarded(setup, call)


# ----------------------------------------------------------------------------- a6-a8
def _packed_prefix(st):
    """the written part of a packed cloud: 12 * offsets[B] bytes"""
    xyz, off = st[3], st[4]
    total = int(off.view(torch.int64)[-1])
    return [xyz[: 12 * total]]


@pytest.mark.parametrize("W,H,s,r,labels", [(37, 13, 4, 2, 48), (21, 11, 2, 3, 90), (13, 9, 8, 1, 500),
                                            (11, 7, 3, 2, 40), (9, 6, 16, 1, 511)])
def test_guard_jbu_compact(W, H, s, r, labels):
    """JBU (vector / scalar kernels, the precise path for wide label ranges), the
    fused count, the scan and the packed write."""
    rng = np.random.default_rng(W * s + r)
    B = 2
    lo = rng.integers(0, labels, size=(B, H, W)).astype(np.int32)
    guide = np.stack([synthgen.value_noise_rgb(b + s, W * s, H * s) for b in range(B)])
    Q = np.ascontiguousarray(P.q_matrix(900.0, 880.0, W * s / 2, H * s / 2, 0.5).reshape(16))
    Wh, Hh = W * s, H * s
    ws = int(P.lib().compact_workspace_bytes(B, Wh, Hh))

    def setup(ar):
        return (ar.add(lo.nbytes, lo), ar.add(guide.nbytes, guide), ar.add(B * Hh * Wh * 4, kind="out"),
                ar.add(B * Hh * Wh * 12, kind="xyz"), ar.add((B + 1) * 8, kind="out"), ar.add(B * 8, kind="out"),
                ar.add(ws, kind="scratch"))

    def call(st):
        l, g, hi, xyz, off, nv, w = st
        assert P.lib().jbu_compact_batch(B, _ptr(l), W, H, _ptr(g), s, 0.9 * s, 15.0, r, Q.ctypes.data_as(C.c_void_p),
                                         1.0, _ptr(hi), _ptr(xyz), B * Hh * Wh, _ptr(off), _ptr(nv), _ptr(w), ws,
                                         _stream()) == 0

    run_guarded(setup, call, post=_packed_prefix)


@pytest.mark.parametrize("W,H,s,r", [(37, 13, 4, 2), (21, 11, 2, 3), (11, 7, 3, 2)])
def test_guard_jbu_reproject_dense(W, H, s, r):
    rng = np.random.default_rng(W + r)
    B = 2
    lo = rng.integers(0, 40, size=(B, H, W)).astype(np.int32)
    guide = np.stack([synthgen.value_noise_rgb(b + 7, W * s, H * s) for b in range(B)])
    Q = np.ascontiguousarray(P.q_matrix(900.0, 880.0, W * s / 2, H * s / 2, 0.5).reshape(16))
    Wh, Hh = W * s, H * s

    def setup(ar):
        return (ar.add(lo.nbytes, lo), ar.add(guide.nbytes, guide), ar.add(B * Hh * Wh * 4, kind="out"),
                ar.add(B * Hh * Wh * 12, kind="out"), ar.add(B * 8, kind="out"))

    def call(st):
        l, g, hi, xyz, nv = st
        assert P.lib().jbu_reproject_batch(B, _ptr(l), W, H, _ptr(g), s, 2.5, 20.0, r, Q.ctypes.data_as(C.c_void_p),
                                           1.0, _ptr(hi), _ptr(xyz), _ptr(nv), _stream()) == 0

    run_guarded(setup, call)


def test_guard_compact_standalone_and_summary():
    B, W, H = 3, 173, 61
    rng = np.random.default_rng(9)
    d = rng.uniform(-1.0, 100.0, size=(B, H, W)).astype(np.float32)
    lo = rng.integers(0, 64, size=(B, 20, 30)).astype(np.int32)
    Q = np.ascontiguousarray(P.q_matrix(900.0, 880.0, W / 2, H / 2, 0.5).reshape(16))
    ws = int(P.lib().compact_workspace_bytes(B, W, H))

    def setup(ar):
        return (ar.add(d.nbytes, d), ar.add(B * H * W * 12, kind="xyz"), ar.add((B + 1) * 8, kind="out"),
                ar.add(B * 8, kind="out"), ar.add(ws, kind="scratch"), ar.add(lo.nbytes, lo), ar.add(B * 64, kind="out"))

    def call(st):
        dd, xyz, off, nv, w, l, summ = st
        assert P.lib().compact_cloud_batch(B, _ptr(dd), W, H, Q.ctypes.data_as(C.c_void_p), 1.0, _ptr(xyz), B * H * W,
                                           _ptr(off), _ptr(nv), _ptr(w), ws, _stream()) == 0
        assert P.lib().pair_summary_batch(B, _ptr(l), 30, 20, _ptr(nv), 7, _ptr(summ), _stream()) == 0

    run_guarded(setup, call, post=lambda st: _packed_prefix((None, None, None, st[1], st[2])))


# ----------------------------------------------------------------------------- f3, f4
def test_guard_features():
    W, H, n, gc, gr, K = 97, 61, 2, 5, 4, 4
    imgs = np.stack([np.asarray(synthgen.iid_gray(i, W, H)) for i in range(n)])
    imgs2 = np.roll(imgs, 3, axis=2)

    def setup(ar):
        return (ar.add(imgs.nbytes, imgs), ar.add(imgs2.nbytes, imgs2), ar.add(n * H * W * 8, kind="out"),
                ar.add(n * gr * gc * K * 8, kind="out"), ar.add(n * gr * gc * K * 8, kind="out"),
                ar.add(n * gr * gc * 4, kind="out"), ar.add(n * gr * gc * K * 8, kind="out"),
                ar.add(n * gr * gc * K * 8, kind="out"))

    def call(st):
        a, b, R25, xy, resp, cnt, match, cost = st
        L = P.lib()
        assert L.harris_corners_batch(n, _ptr(a), W, H, gc, gr, K, 1, _ptr(R25), _ptr(xy), _ptr(resp), _ptr(cnt),
                                      _stream()) == 0
        assert L.zssd_match_batch(n, _ptr(a), _ptr(b), W, H, _ptr(xy), gr * gc * K, 3, 8, 2 ** 62, _ptr(match),
                                  _ptr(cost), _stream()) == 0

    run_guarded(setup, call)


def test_guard_icp():
    rng = np.random.default_rng(3)
    tgt = rng.uniform(-1, 1, size=(3001, 3)).astype(np.float32)
    src = (tgt + np.float32([0.01, -0.02, 0.015])).astype(np.float32)
    src[::97] = np.nan
    ns, nt = src.shape[0], tgt.shape[0]
    init = (C.c_double * 12)(1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0)
    ws = int(P.lib().icp_workspace_bytes(ns, nt))

    def setup(ar):
        return ar.add(src.nbytes, src), ar.add(tgt.nbytes, tgt), ar.add(ws, kind="scratch"), ar.add(16 * 8, kind="out")

    def call(st):
        s_, t_, w, o = st
        assert P.lib().icp_register(_ptr(s_), ns, _ptr(t_), nt, init, 10, 0.2, 1e-6, 1, _ptr(w), ws, _ptr(o),
                                    _stream()) == 0

    run_guarded(setup, call)


def test_guard_video_generator():
    from synthgen import video
    sc = video.VideoScene(3, 100, 36, 4, 8, 48)

    def setup(ar):
        return ar.add(3 * 36 * 100 * 3, kind="out")

    def call(o):
        video.frames_device(sc, 5, t(o, torch.uint8, (3, 36, 100, 3)))

    run_guarded(setup, call)
