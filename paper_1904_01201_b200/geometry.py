"""Planar helpers and the device-resident SegmentIndex facade.

Drop-in for /root/reference/pkg/src/navsim/geometry.py's hot-path surface:
``wrap_angle`` (:19-24), ``segment_normals`` (:66-73) and ``SegmentIndex``
(:100-206) whose ``raycast`` / ``raycast_brute`` / ``cast_disc`` /
``clearance`` run as CUDA kernels (nv_raycast / nv_cast_disc / nv_clearance
in include/navsim_b200.h).  The uniform grid is built by the C ABI exactly
like SegmentIndex.__init__ and lives in HBM.
"""
from __future__ import annotations

import math

import numpy as np

from . import _native as nat
from .scene import IDENTITY, Transform2D  # noqa: F401  (re-export, geometry.py:27)


def wrap_angle(theta: float) -> float:
    """Wrap to (-pi, pi] (geometry.py:19-24)."""
    out = math.fmod(theta + math.pi, 2.0 * math.pi)
    if out <= 0.0:
        out += 2.0 * math.pi
    return out - math.pi


def segment_lengths(segs) -> np.ndarray:
    s = np.asarray(segs, dtype=np.float64)
    return np.hypot(s[:, 2] - s[:, 0], s[:, 3] - s[:, 1])


def segment_normals(segs) -> np.ndarray:
    """Unit left normals (n, 2); zero-length segments give zeros."""
    s = np.asarray(segs, dtype=np.float64).reshape(-1, 4)
    ex, ey = s[:, 2] - s[:, 0], s[:, 3] - s[:, 1]
    ln = np.hypot(ex, ey)
    ln = np.where(ln > 0.0, ln, 1.0)
    return np.stack([-ey / ln, ex / ln], axis=1)


def _upload_scene(ctx, segs, sem, albedo, wall_h, floor3, ceil3):
    segs = np.ascontiguousarray(segs, dtype=np.float64).reshape(-1, 4)
    sem = np.ascontiguousarray(sem, dtype=np.uint16)
    albedo = np.ascontiguousarray(albedo, dtype=np.float64).reshape(-1, 3)
    f3 = np.ascontiguousarray(floor3, dtype=np.float64)
    c3 = np.ascontiguousarray(ceil3, dtype=np.float64)
    nat.check(ctx.lib.nv_scene_upload(ctx.handle, nat.ptr(segs), nat.ptr(sem), nat.ptr(albedo),
                                      len(segs), float(wall_h), nat.ptr(f3), nat.ptr(c3)))


class SegmentIndex:
    """Uniform 1 m grid over world segments, resident on the GPU."""

    CELL = 1.0

    def __init__(self, segs, device: int = 0, _ctx=None):
        s = np.asarray(segs, dtype=np.float64).reshape(-1, 4)
        self.segs = s
        self.ax, self.ay = np.ascontiguousarray(s[:, 0]), np.ascontiguousarray(s[:, 1])
        self.bx, self.by = np.ascontiguousarray(s[:, 2]), np.ascontiguousarray(s[:, 3])
        self.ex, self.ey = self.bx - self.ax, self.by - self.ay
        if _ctx is None:
            _ctx = nat.Context(device)
            _upload_scene(_ctx, s, np.zeros(len(s), np.uint16), np.zeros((len(s), 3)), 2.5,
                          (0, 0, 0), (0, 0, 0))
        self._ctx = _ctx
        import ctypes
        x0, y0 = ctypes.c_double(), ctypes.c_double()
        nx, ny, ni = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        nat.check(_ctx.lib.nv_scene_grid_info(_ctx.handle, ctypes.byref(x0), ctypes.byref(y0),
                                              ctypes.byref(nx), ctypes.byref(ny), ctypes.byref(ni)))
        self.x0, self.y0, self.nx, self.ny = x0.value, y0.value, nx.value, ny.value
        self.n_items = ni.value

    def __len__(self) -> int:
        return len(self.segs)

    @property
    def context(self):
        return self._ctx

    def _dev(self, a, dtype=None):
        import torch
        return torch.as_tensor(np.ascontiguousarray(a), device=f"cuda:{self._ctx.device}",
                               dtype=dtype)

    def raycast(self, origin, dirs, t_max: float = 1e9, brute: bool = False):
        """Nearest hit per ray (raycast_grid, _kernels.py:51); t in units of dir."""
        import torch
        d = np.asarray(dirs, dtype=np.float64).reshape(-1, 2)
        m = len(d)
        dev = f"cuda:{self._ctx.device}"
        ox = torch.full((m,), float(origin[0]), dtype=torch.float64, device=dev)
        oy = torch.full((m,), float(origin[1]), dtype=torch.float64, device=dev)
        dx, dy = self._dev(d[:, 0]), self._dev(d[:, 1])
        t = torch.empty(m, dtype=torch.float64, device=dev)
        i = torch.empty(m, dtype=torch.int64, device=dev)
        nat.check(self._ctx.lib.nv_raycast(self._ctx.handle, nat.ptr(ox), nat.ptr(oy), nat.ptr(dx),
                                           nat.ptr(dy), m, float(t_max), int(brute), nat.ptr(t),
                                           nat.ptr(i), nat.stream_handle(dev)))
        return t.cpu().numpy(), i.cpu().numpy()

    def raycast_brute(self, origin, dirs):
        """Exhaustive scan (raycast_all, _kernels.py:16)."""
        return self.raycast(origin, dirs, brute=True)

    def cast_disc_batch(self, px, py, ux, uy, radius):
        """Batched disc casts on device tensors/arrays -> (t, seg, tan (m,2))."""
        import torch
        dev = f"cuda:{self._ctx.device}"
        cols = [self._dev(np.asarray(v, dtype=np.float64).reshape(-1)) for v in (px, py, ux, uy, radius)]
        m = cols[0].numel()
        t = torch.empty(m, dtype=torch.float64, device=dev)
        seg = torch.empty(m, dtype=torch.int64, device=dev)
        tan = torch.empty((m, 2), dtype=torch.float64, device=dev)
        nat.check(self._ctx.lib.nv_cast_disc(self._ctx.handle, *(nat.ptr(c) for c in cols), m,
                                             nat.ptr(t), nat.ptr(seg), nat.ptr(tan),
                                             nat.stream_handle(dev)))
        return t.cpu().numpy(), seg.cpu().numpy(), tan.cpu().numpy()

    def cast_disc(self, pos, motion, radius: float):
        """First contact of a swept disc (geometry.py:183-192)."""
        t, seg, tan = self.cast_disc_batch([pos[0]], [pos[1]], [motion[0]], [motion[1]], [radius])
        return float(t[0]), int(seg[0]), tan[0].copy()

    def clearance_batch(self, px, py, search_radius: float = 2.0):
        import torch
        dev = f"cuda:{self._ctx.device}"
        x = self._dev(np.asarray(px, dtype=np.float64).reshape(-1))
        y = self._dev(np.asarray(py, dtype=np.float64).reshape(-1))
        out = torch.empty(x.numel(), dtype=torch.float64, device=dev)
        nat.check(self._ctx.lib.nv_clearance(self._ctx.handle, nat.ptr(x), nat.ptr(y), x.numel(),
                                             float(search_radius), nat.ptr(out),
                                             nat.stream_handle(dev)))
        return out.cpu().numpy()

    def clearance(self, pos, search_radius: float = 2.0) -> float:
        """Distance to the nearest segment (geometry.py:194-206)."""
        return float(self.clearance_batch([pos[0]], [pos[1]], search_radius)[0])


def navigable_mask(segs, bounds, resolution: float, agent_radius: float):
    """geometry.navigable_mask (geometry.py:209-250): (mask, origin of cell
    (0, 0)'s center, per-cell wall distance), built on the device
    (nav.rasterize_navigable -> nv_nav_build)."""
    from .nav import rasterize_navigable
    grid = rasterize_navigable(segs, bounds, resolution, agent_radius)
    return grid.navigable, np.asarray(grid.origin, dtype=np.float64), grid.clearance
