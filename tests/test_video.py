"""The synthetic UAV video of the C5 stream (synthgen/video.py, synthgen/synth_video.cu):
input generation only -- checked for the structure the workload needs (consecutive
frames are virtual stereo pairs with the scene's disparities), for
determinism, and (-m gpu) for bit-equality of the device generator with its numpy
twin."""
import numpy as np
import pytest
import torch

from synthgen.video import VideoScene, frames_device


def test_consecutive_frames_are_a_stereo_pair():
    """right(x - s*d) = left(x) between frames k and k+1 for (nearly) every pixel of
    frame k whose world point stays visible; labels inside [dmin, dmax]."""
    sc = VideoScene(5, 512, 256, 4, 8, 48)
    for k in (0, 3, 250):
        f0, f1 = sc.frame(k), sc.frame(k + 1)
        lab, X = sc.visible(k)
        lab1, X1 = sc.visible(k + 1)
        vis = lab >= 0
        assert vis.mean() > 0.97
        assert lab[vis].min() >= 8 and lab[vis].max() <= 48
        ys, xs = np.nonzero(vis)
        xr = xs - 4 * lab[ys, xs]
        ok = xr >= 0
        ys, xs, xr = ys[ok], xs[ok], xr[ok]
        same_point = X1[ys, xr] == X[ys, xs]  # still visible in frame k+1 (not occluded)
        assert same_point.mean() > 0.95
        assert np.array_equal(f1[ys[same_point], xr[same_point]], f0[ys[same_point], xs[same_point]])


def test_video_is_deterministic_and_textured():
    a = VideoScene(9, 256, 128, 4, 8, 48)
    b = VideoScene(9, 256, 128, 4, 8, 48)
    c = VideoScene(10, 256, 128, 4, 8, 48)
    fa, fb, fc = a.frame(7), b.frame(7), c.frame(7)
    assert np.array_equal(fa, fb) and not np.array_equal(fa, fc)
    assert fa.std() > 20  # texture survives the 4x box mean
    grey = fa.astype(np.float64).mean(axis=2).reshape(32, 4, 64, 4).mean(axis=(1, 3))
    assert grey.std() > 10
    assert np.array_equal(a.frame(7, rows=[0, 50, 127]), fa[[0, 50, 127]])


def test_labels_lo_matches_visible_footprints():
    sc = VideoScene(3, 256, 128, 4, 16, 40)
    lo = sc.labels_lo(2)
    lab, _ = sc.visible(2)
    assert lo.shape == (32, 64)
    assert np.array_equal(lo, lab[::4, ::4])


@pytest.mark.gpu
@pytest.mark.parametrize("W,H,s,dmin,dmax,k0,n", [(256, 128, 4, 8, 48, 0, 3), (200, 96, 2, 16, 96, 4000, 2),
                                                  (64, 40, 8, 0, 12, 77, 4)])
def test_device_generator_equals_numpy_twin(W, H, s, dmin, dmax, k0, n):
    sc = VideoScene(1234 + W, W, H, s, dmin, dmax)
    out = torch.empty((n, H, W, 3), dtype=torch.uint8, device="cuda")
    frames_device(sc, k0, out)
    got = out.cpu().numpy()
    for i in range(n):
        assert np.array_equal(got[i], sc.frame(k0 + i)), (k0 + i)


@pytest.mark.gpu
def test_device_generator_full_frame_rows():
    """A 2.7K frame deep into the 4096-pair stream: sampled rows equal the twin."""
    sc = VideoScene(1902, 2704, 1520, 4, 8, 48)
    out = torch.empty((1, 1520, 2704, 3), dtype=torch.uint8, device="cuda")
    frames_device(sc, 4095, out)
    rows = [0, 3, 511, 760, 1519]
    assert np.array_equal(out[0, rows].cpu().numpy(), sc.frame(4095, rows=rows))
