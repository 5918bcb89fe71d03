"""Bit-exact numpy model of the frame writers' packed-f16 RGB shading
(paper_1904_01201_b200/csrc/fill.cuh shade_pair, navsim_b200.cu
build_camera_tables / nv_scene_upload), and the reference formula it
approximates (fill_frame, /root/reference/pkg/src/navsim/_kernels.py:171-207):

    reference   rgb = albedo * (0.2 + 0.8 * cos_a)           (f64, in [0, 1])
    device      t   = fma_f16(num16, inv16, f16(0.2))         num16 = f16(f32(0.8) * f32(|d.n|))
                u8  = fma_f16(col16, t, 1024) - 1024          col16 = f16(f32(albedo * 255))
                                                              inv16 = f16(f32(1 / |(d, v)|))

An fma.rn.f16 is one rounding of the exact a*b + c: the product of two f16
values is exact in f64 and, at these magnitudes, so is the sum, so
rounding the f64 result to f16 once (numpy, round-to-nearest-even) is the
hardware result.  tests/test_gpu_shading_model.py checks the model against
the device bit for bit.
"""
import numpy as np

H2_POINT2 = float(np.float16(0.2))  # the f16 constant 0.2 of fill.cuh (NV_H2_POINT2)


def f16(x):
    return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def fma16(a, b, c):
    """fma.rn.f16: a, b, c are f16 values (as f64)."""
    return f16(np.asarray(a) * np.asarray(b) + np.asarray(c))


def shade_u8(col16, num16, inv16):
    """Device u8 channel value from the f16 inputs."""
    t = fma16(num16, inv16, H2_POINT2)
    return fma16(col16, t, 1024.0) - 1024.0


def col16_of(albedo):
    return f16(f32(np.asarray(albedo, dtype=np.float64) * 255.0))


def num16_of(dot_abs):
    """0.8 * |cos numerator| as the writers pack it: f32 product, then f16."""
    return f16(f32(np.float32(0.8) * f32(dot_abs)))


def inv16_of(u, v):
    """Shading-table entry 1 / sqrt(1 + u^2 + v^2) (f64 -> f32 -> f16)."""
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    return f16(f32(1.0 / np.sqrt(1.0 + u * u + v * v)))


def f16_codes(lo, hi):
    """Every non-negative f16 value in [lo, hi] (as f64), ascending."""
    bits = np.arange(0, 0x7C00, dtype=np.uint16)
    v = bits.view(np.float16).astype(np.float64)
    return v[(v >= lo) & (v <= hi)]


def half_ulp(v16):
    """Half the spacing of the f16 grid at each value (the rounding radius)."""
    v = np.asarray(v16, dtype=np.float64)
    with np.errstate(over="ignore"):
        up = np.nextafter(v.astype(np.float16), np.float16(np.inf)).astype(np.float64)
    up = np.where(np.isfinite(up), up, 2.0 * v - np.nextafter(v.astype(np.float16), np.float16(0))
                  .astype(np.float64))  # the largest finite f16: the spacing below it
    return (up - v) * 0.5


def render_rgb_model(t_col, i_col, dirx, diry, H, focal, cam_h, wall_h, max_range, nx, ny,
                     albedo, floor_color, ceil_color):
    """The device RGB frames (u8 [n, H, W, 3]) for given column hits, from the
    same f64 / f32 / f16 steps as the device path (column epilogue row
    classification, RowRec / ColRec packing, shade_pair)."""
    t_col = np.asarray(t_col, dtype=np.float64)
    n, W = t_col.shape
    j = np.arange(W, dtype=np.float64)
    u = ((j + 0.5) - W * 0.5) / focal
    i = np.arange(H, dtype=np.float64)
    v = (H * 0.5 - (i + 0.5)) / focal
    inv = inv16_of(u[None, :], v[:, None])                        # [H, W]
    with np.errstate(divide="ignore"):
        tc = np.where(v > 0, (wall_h - cam_h) / v, np.inf)
        tf = np.where(v < 0, -cam_h / v, np.inf)
    # per-row plane records (ceiling rows v > 0, floor rows v < 0; void beyond range)
    plane_t = np.where(v > 0, tc, np.where(v < 0, tf, np.inf))
    plane_lit = plane_t < max_range
    plane_col = np.where((v > 0)[:, None], np.asarray(ceil_color)[None, :],
                         np.asarray(floor_color)[None, :])            # [H, 3]
    plane_col16 = np.where(plane_lit[:, None], col16_of(plane_col), 0.0)
    plane_num16 = np.where(plane_lit, num16_of(np.abs(v)), 0.0)
    out = np.zeros((n, H, W, 3), dtype=np.uint8)
    for e in range(n):
        s = t_col[e]
        k = np.asarray(i_col[e], dtype=np.int64)
        dx, dy = np.asarray(dirx[e], dtype=np.float64), np.asarray(diry[e], dtype=np.float64)
        lit = (s < max_range) & (k >= 0)
        kk = np.where(k >= 0, k, 0)
        dot = np.abs(dx * nx[kk] + dy * ny[kk])
        wall_num16 = np.where(lit, num16_of(dot), 0.0)                 # [W]
        wall_col16 = np.where(lit[:, None], col16_of(albedo[kk]), 0.0)  # [W, 3]
        ceil_px = tc[:, None] <= s[None, :]                            # rows i < lo
        floor_px = tf[:, None] <= s[None, :]                           # rows i >= hi
        band = ~(ceil_px | floor_px)
        num = np.where(band, wall_num16[None, :], plane_num16[:, None])
        for c in range(3):
            col = np.where(band, wall_col16[None, :, c], plane_col16[:, c][:, None])
            out[e, :, :, c] = shade_u8(col, num, inv).astype(np.uint8)
    return out
