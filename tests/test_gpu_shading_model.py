"""The device's packed-f16 RGB shading equals the numpy model of
tests/f16_shading.py bit for bit (the model the exhaustive bound of
tests/test_shading_f16_bound.py is proven on), through fill_frame's
operator entry (nv_fill_frames, _kernels.py:128-207) with adversarial
inputs: albedos at 0, 1 and on f16 rounding boundaries of albedo*255,
extreme floor / ceiling colours, random wall normals and headings, misses,
hits beyond max_range, for both frame writers (warp-specialised TMA writer
and the per-pixel kernel) and two aspect ratios.
"""
import math

import numpy as np
import pytest

from f16_shading import render_rgb_model

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_01201_b200 as nb
    from paper_1904_01201_b200 import _native
    _native.load()
    return nb


def _adversarial_albedo(rng, n):
    # albedo*255 at f16 rounding midpoints (spacing 0.125 on [128, 256)), the
    # extremes, and uniform values
    mids = (np.arange(1024, 2040) * 0.125 + 0.0625) / 255.0
    base = np.concatenate([[0.0, 1.0, 1.0 - 1e-12, 1e-12, 0.5, 254.5 / 255, 0.5 / 255], mids])
    vals = np.concatenate([base, rng.uniform(0, 1, 3 * n)])
    return np.clip(rng.choice(vals, size=(n, 3)), 0.0, 1.0)


@pytest.mark.parametrize("W,H", [(256, 64), (128, 128)])
@pytest.mark.parametrize("fill_mode", ["auto", "generic"])
def test_device_rgb_equals_f16_model(nb, W, H, fill_mode):
    from paper_1904_01201_b200 import _native as nat
    rng = np.random.default_rng(7 + W + H)
    n_seg = 4000
    a = rng.uniform(-20, 20, (n_seg, 2))
    ang = rng.uniform(-math.pi, math.pi, n_seg)
    ln = rng.uniform(0.05, 3.0, n_seg)
    segs = np.column_stack([a, a + ln[:, None] * np.column_stack([np.cos(ang), np.sin(ang)])])
    alb = _adversarial_albedo(rng, n_seg)
    sem = rng.integers(1, 60000, n_seg).astype(np.uint16)
    floor_c, ceil_c = (1.0, 0.0, 254.5 / 255.0), (1e-12, 1.0, 0.5)
    focal = (W * 0.5) / math.tan(math.radians(90.0) * 0.5)
    suite = (nb.SensorConfig("rgb", W, H),)
    sim = nb.BatchSimulator(segs, sem, alb, 1, sensor_configs=suite, floor_color=floor_c,
                            ceiling_color=ceil_c)
    c = sim.ctx
    nat.check(c.lib.nv_set_fill_mode(c.handle, nat.NV_FILL_AUTO if fill_mode == "auto"
                                     else nat.NV_FILL_GENERIC))
    n = 24
    # column hits: distances incl. misses (inf) and hits beyond max_range,
    # directions = the camera's columns at random headings (unit forward)
    t_col = rng.uniform(0.02, 12.0, (n, W))
    t_col[rng.random((n, W)) < 0.05] = np.inf
    i_col = rng.integers(0, n_seg, (n, W)).astype(np.int64)
    i_col[~np.isfinite(t_col)] = -1
    hd = rng.uniform(-math.pi, math.pi, n)
    j = np.arange(W, dtype=np.float64)
    u = ((j + 0.5) - W * 0.5) / focal
    ch, sh = np.cos(hd)[:, None], np.sin(hd)[:, None]
    dirx = ch + u[None, :] * sh
    diry = sh + u[None, :] * (-ch)
    ex, ey = segs[:, 2] - segs[:, 0], segs[:, 3] - segs[:, 1]
    hyp = np.hypot(ex, ey)
    nx, ny = -ey / hyp, ex / hyp
    dev = {k: torch.as_tensor(np.ascontiguousarray(v), device="cuda:0")
           for k, v in (("t", t_col), ("i", i_col), ("dx", dirx), ("dy", diry))}
    rgb = torch.empty((n, H, W, 3), dtype=torch.uint8, device="cuda:0")
    nat.check(c.lib.nv_fill_frames(c.handle, 0, n, nat.ptr(dev["t"]), nat.ptr(dev["i"]),
                                   nat.ptr(dev["dx"]), nat.ptr(dev["dy"]), 1.5, nat.ptr(rgb),
                                   None, None, nat.stream_handle("cuda:0")))
    torch.cuda.synchronize()
    want = render_rgb_model(t_col, i_col, dirx, diry, H, focal, 1.5, 2.5, 10.0, nx, ny, alb,
                            floor_c, ceil_c)
    got = rgb.cpu().numpy()
    bad = np.argwhere(got != want)
    assert len(bad) == 0, f"{len(bad)} channel values differ, first {bad[:3]}"
