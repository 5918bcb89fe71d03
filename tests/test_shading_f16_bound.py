"""Exhaustive error bound of the packed-f16 RGB shading against the reference's
f64 fill_frame formula (/root/reference/pkg/src/navsim/_kernels.py:171-207),
on the north-star tolerance grid (RGB within 1/255 per channel).

The device computes (tests/f16_shading.py, bit-exact model of fill.cuh):
    t   = fma_f16(num16, inv16, f16(0.2)),   u8 = fma_f16(col16, t, 1024) - 1024
from three f16-rounded inputs: num16 ~ 0.8 |d.n| (or 0.8 |v| on planes),
inv16 ~ 1/|(d, v)|, col16 ~ albedo * 255.  The reference's value in u8
units is albedo*255 * (0.2 + 0.8 |d.n| / |(d, v)|).

The sweep is exhaustive over the f16 grid, with each input's exact value
anywhere in its f16 rounding interval:
  1. every (inv16, num16) pair an actual pixel can produce -- inv16 every f16
     in [2^-14, 1] (|(d, v)| up to 16384: e.g. hfov 179 deg at aspect 1:100),
     num16 every f16 with
     num16 * inv16 <= 0.8 (1 + slack), i.e. cos <= 1 -- gives t16 and the
     hull of the true t over the pair's rounding box (clipped to cos <= 1);
  2. every col16 (every f16 in [0, 255]) against every reachable t16: the
     error is linear in the exact albedo and t, so its maximum over the
     (albedo, t) box is at a corner.
The worst case is printed and must stay below one 8-bit step.
"""
import numpy as np

from f16_shading import H2_POINT2, f16, f16_codes, fma16, half_ulp

# relative slack for the f32 step each input takes before its f16 rounding
# (f64 -> f32 -> f16; the f32 rounding error is < 2^-24 relative)
F32_SLACK = 2.0 ** -23


def _t_hull():
    """{t16: (min true t, max true t)} over every reachable (num16, inv16)."""
    inv_all = f16_codes(2.0 ** -14, 1.0)
    num_all = f16_codes(0.0, 65504.0)
    hn_all = half_ulp(num_all) + num_all * F32_SLACK
    t_lo = {}
    t_hi = {}
    for inv in inv_all:
        hi_inv = inv + float(half_ulp(inv)) + inv * F32_SLACK
        lo_inv = max(inv - float(half_ulp(inv)) - inv * F32_SLACK, 0.0)
        # reachable: some exact (num, inv) in the box has num * inv <= 0.8
        ok = (num_all - hn_all) * lo_inv <= 0.8
        num = num_all[ok]
        hn = hn_all[ok]
        t16 = fma16(num, inv, H2_POINT2)
        tl = 0.2 + np.maximum(num - hn, 0.0) * lo_inv
        th = np.minimum(0.2 + (num + hn) * hi_inv, 1.0)
        # t16 is non-decreasing in num: reduce over runs of equal t16
        edges = np.flatnonzero(np.diff(t16)) + 1
        starts = np.concatenate([[0], edges])
        keys = t16[starts]
        lo_r = np.minimum.reduceat(tl, starts)
        hi_r = np.maximum.reduceat(th, starts)
        for k, a, b in zip(keys.tolist(), lo_r.tolist(), hi_r.tolist()):
            if k in t_lo:
                t_lo[k] = min(t_lo[k], a)
                t_hi[k] = max(t_hi[k], b)
            else:
                t_lo[k] = a
                t_hi[k] = b
    keys = np.array(sorted(t_lo))
    return keys, np.array([t_lo[k] for k in keys]), np.array([t_hi[k] for k in keys])


def test_f16_shading_error_below_one_step():
    t16, tlo, thi = _t_hull()
    assert t16.min() >= H2_POINT2 and t16.max() <= 1.0 + 2.0 ** -10
    col16 = f16_codes(0.0, 255.0)
    hc = half_ulp(col16) + col16 * F32_SLACK
    clo = np.maximum(col16 - hc, 0.0)
    chi = np.minimum(col16 + hc, 255.0)
    worst, arg = -1.0, None
    for k in range(len(t16)):
        dev = fma16(col16, t16[k], 1024.0) - 1024.0
        err = np.maximum(np.abs(dev - clo * tlo[k]), np.abs(dev - chi * thi[k]))
        m = int(np.argmax(err))
        if err[m] > worst:
            worst, arg = float(err[m]), (float(col16[m]), float(t16[k]), float(tlo[k]),
                                         float(thi[k]), float(dev[m]))
    print(f"\nworst |device - reference| = {worst:.4f} of one 8-bit step "
          f"(col16={arg[0]}, t16={arg[1]}, true t in [{arg[2]:.6f}, {arg[3]:.6f}], "
          f"device u8={arg[4]:.0f}); {len(t16)} reachable t16 values x {len(col16)} col16 values")
    assert worst < 1.0


def test_model_is_exact_on_the_f16_grid():
    """Sanity of the model itself: with exact f16 inputs and no rounding
    slack the device value is the round-to-nearest of col16 * t16."""
    col = f16_codes(0.0, 255.0)[::37]
    for t in (H2_POINT2, 0.5, 0.75, 1.0):
        dev = fma16(col, t, 1024.0) - 1024.0
        assert np.all(np.abs(dev - col * t) <= 0.5)
        assert np.array_equal(dev, f16(np.rint(col * t) + 1024.0) - 1024.0)
