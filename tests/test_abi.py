"""C-ABI library checks that need no GPU (-m "not gpu"): the library loads, exports
every symbol include/vsbp.h declares, validates arguments and quantises parameters
the same way as the (independently written) oracle; compute entry points fail
loudly without a GPU (there is no CPU fallback)."""
import ctypes as C
import os
import re

import pytest
import torch

import oracle
import paper_1902_09733_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "vsbp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    lib = P.lib()
    names = declared_symbols()
    assert len(names) >= 20, names
    for n in names:
        assert hasattr(lib, n), f"libvsbp.so does not export {n}"
    assert set(names) == set(P._EXPORTS), "binding and header disagree"


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("case", [
    (0.07, 15.0, 1.7), (0.5, 2.5, 1.25), (0.0, 1.0, 0.01), (0.0112, 15.0, 4.0), (1.0, 30.0, 3.0)])
def test_quantisation_matches_oracle(case):
    h = C.c_void_p()
    assert P.lib().bp_create(64, 48, 16, 1, 5, *case, C.byref(h)) == 0
    out = (C.c_int32 * 8)()
    assert P.lib().bp_get_params(h, out) == 0
    q = oracle.quantize(*case)
    assert list(out)[:4] == [q.lam_q, q.tau_d, q.tau_q, q.S]
    assert out[4] == (1 if q.tau_q <= 255 else 2 if q.tau_q <= 65535 else 4)
    P.lib().bp_destroy(h)


def test_create_rejects():
    h = C.c_void_p()
    L = P.lib()
    assert L.bp_create(0, 48, 16, 1, 5, 0.07, 15.0, 1.7, C.byref(h)) == -1
    assert L.bp_create(64, 48, 1, 1, 5, 0.07, 15.0, 1.7, C.byref(h)) == -1
    assert L.bp_create(64, 48, 16, 0, 5, 0.07, 15.0, 1.7, C.byref(h)) == -1
    assert L.bp_create(64, 48, 16, 1, 0, 0.07, 15.0, 1.7, C.byref(h)) == -1
    assert L.bp_create(64, 48, 16, 1, 5, -1.0, 15.0, 1.7, C.byref(h)) == -1
    assert L.bp_create(64, 48, 16, 1, 5, 0.07, 0.4, 1.7, C.byref(h)) == -1
    # R-25: both sides reject the same overflow
    assert L.bp_create(4, 4, 4, 12, 1, 1000.0, 255.0, 1.7, C.byref(h)) == -3
    with pytest.raises(oracle.OracleError):
        import numpy as np
        img = np.zeros((4, 4), np.uint8)
        oracle.bp_disparity(img, img, 4, 12, 1, lam=1000.0, data_trunc=255.0)


def test_level_dims_and_workspace():
    h = C.c_void_p()
    L = P.lib()
    assert L.bp_create(676, 380, 64, 5, 5, 0.07, 15.0, 1.7, C.byref(h)) == 0
    dims = []
    for l in range(5):
        w, hh = C.c_int(), C.c_int()
        assert L.bp_level_dims(h, l, C.byref(w), C.byref(hh)) == 0
        dims.append((w.value, hh.value))
    assert dims == oracle.level_dims(676, 380, 5)
    n1p = L.bp_workspace_bytes(h, 1)  # default: two iterations per launch -> a second u8 message array per level
    assert L.bp_set_option(h, P.VSBP_OPT_PAIR, 0) == 0
    n1 = L.bp_workspace_bytes(h, 1)
    n4 = L.bp_workspace_bytes(h, 4)
    assert n1 > 0 and n4 >= 4 * n1 - 4096 * 10
    msgs = sum(8 * h_ * ((w_ + 1) // 2) * 64 for w_, h_ in dims if w_ * h_ >= 100000)  # one u8 array per large level
    assert msgs - 256 * 5 <= n1p - n1 <= msgs + 256 * 5
    # u16-cost levels (level 1 here: 338 x 190 = 64K px, level 2: 169 x 95 = 16K px)
    # get the second array only when the batch holds >= 2M of their pixels (32 / 125
    # pairs) and they have >= 10K px (level 3: 4K, never); u8 levels from 100K px
    mm = [8 * hh * ((w + 1) // 2) * 64 for w, hh in dims]
    for B, fused in ((31, ()), (32, (1,)), (124, (1,)), (125, (1, 2))):
        base = L.bp_workspace_bytes(h, B)
        assert L.bp_set_option(h, P.VSBP_OPT_PAIR, 1) == 0
        extra = L.bp_workspace_bytes(h, B) - base
        assert L.bp_set_option(h, P.VSBP_OPT_PAIR, 0) == 0
        want = B * (msgs + sum(mm[l] for l in fused))
        assert want - 256 * 5 <= extra <= want + 256 * 5, (B, extra, want)
    # message option: narrower than lossless is refused, wider accepted
    assert L.bp_set_option(h, P.VSBP_OPT_MSG_BYTES, 2) == 0
    assert L.bp_workspace_bytes(h, 1) > n1
    assert L.bp_set_option(h, P.VSBP_OPT_MSG_BYTES, 3) == -1
    # 0/1 switches; anything else (or an unknown option) is refused
    for opt, top in ((P.VSBP_OPT_KERNEL, 1), (P.VSBP_OPT_DIMG, 2), (P.VSBP_OPT_FINAL, 3), (P.VSBP_OPT_PAIR, 3)):
        assert all(L.bp_set_option(h, opt, v) == 0 for v in range(top + 1))
        assert L.bp_set_option(h, opt, top + 1) == -1 and L.bp_set_option(h, opt, -1) == -1
    assert L.bp_set_option(h, 99, 0) == -1
    assert L.bp_set_workspace(h, C.c_void_p(256), 10, 1) == -2  # too small
    assert L.bp_disparity_batch(h, 1, C.c_void_p(256), C.c_void_p(256), C.c_void_p(256), None) == -2  # no ws
    L.bp_destroy(h)
    h2 = C.c_void_p()
    assert L.bp_create(64, 48, 16, 1, 5, 0.07, 15.0, 100.0, C.byref(h2)) == 0  # tau_q = 12800 -> u16
    out = (C.c_int32 * 8)()
    L.bp_get_params(h2, out)
    assert out[4] == 2
    assert L.bp_set_option(h2, P.VSBP_OPT_MSG_BYTES, 1) == -1
    L.bp_destroy(h2)


def test_other_entry_points_validate():
    L = P.lib()
    Q = (C.c_double * 16)()
    assert L.reproject_batch(1, C.c_void_p(256), 4, 4, Q, 0.0, C.c_void_p(256), C.c_void_p(256), None) == -1
    assert L.jbu_upsample_batch(1, C.c_void_p(256), 4, 4, C.c_void_p(256), 4, C.c_void_p(256), 1.0, 15.0, 0,
                                None) == -1
    assert L.jbu_upsample_batch(1, C.c_void_p(256), 4, 4, C.c_void_p(256), 4, C.c_void_p(256), 0.0, 15.0, 2,
                                None) == -1
    assert L.prep_downsample_batch(1, C.c_void_p(256), 10, 10, 3, C.c_void_p(256), None) == -2
    # sigma_s so small that the window's weights leave f32 range is refused
    assert L.jbu_upsample_batch(1, C.c_void_p(256), 4, 4, C.c_void_p(256), 4, C.c_void_p(256), 0.2, 15.0, 2,
                                None) == -1
    assert L.vsbp_strerror(-3) == b"int32 fixed-point bound exceeded"


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    """Compute calls on a machine without a GPU fail with VSBP_ECUDA."""
    L = P.lib()
    rc = L.prep_downsample_batch(1, C.c_void_p(256), 8, 8, 2, C.c_void_p(512), None)
    assert rc == -4
    assert b"CUDA" in L.vsbp_strerror(-4)
