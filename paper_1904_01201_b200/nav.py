"""Navigable-space queries at the drop-in boundary (reference: pkg/src/navsim/nav.py).

Same names, arguments and errors as the reference module, computed on the
GPU through the C ABI: ``rasterize_navigable`` builds the occupancy grid and
per-cell wall clearance on the device (nv_nav_build), ``distance_field``
runs the goal's geodesic field on the device (nv_nav_fields, bit-identical to
the reference's Dijkstra), ``geodesic_distance`` interpolates it on the
device (nv_nav_geodesic).  The grid's ``navigable`` / ``clearance`` arrays and
a field's ``dist`` are host copies made on first access, like the reference's
numpy arrays; ``DistanceField.dist_device`` is the resident torch tensor.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat

DEFAULT_RESOLUTION = 0.05   # nav.py:18
SNAP_RADIUS = 0.2           # nav.py:19

__all__ = ["DEFAULT_RESOLUTION", "SNAP_RADIUS", "NavError", "OccupancyGrid", "DistanceField",
           "rasterize_navigable", "distance_field", "distance_fields", "geodesic_distance",
           "sample_navigable"]


class NavError(Exception):
    pass


@dataclass(eq=False)
class OccupancyGrid:
    """Boolean navigability per cell center over a scene's bounds (nav.py:27-62),
    resident on the device of ``ctx``."""

    origin: np.ndarray
    resolution: float
    width: int
    height: int
    ctx: object = field(repr=False)
    _host: dict = field(default_factory=dict, repr=False)
    gen: int = 0  # the context's grid generation this object describes

    def _check(self):
        """The context holds one grid; a rebuild invalidates older grid objects
        (their sizes would no longer match the device buffers)."""
        if getattr(self.ctx, "_nav_gen", 0) != self.gen:
            raise NavError("occupancy grid was rebuilt on its context; use the new grid")

    def _pull(self):
        self._check()
        if not self._host:
            m = np.empty((self.height, self.width), dtype=np.uint8)
            d = np.empty((self.height, self.width), dtype=np.float64)
            nat.check(self.ctx.lib.nv_nav_copy(self.ctx.handle, self.width, self.height,
                                               nat.ptr(m), nat.ptr(d)))
            self._host["navigable"] = m.astype(bool)
            self._host["clearance"] = d
        return self._host

    @property
    def navigable(self) -> np.ndarray:
        return self._pull()["navigable"]

    @property
    def clearance(self) -> np.ndarray:
        return self._pull()["clearance"]

    def cell_of(self, p) -> tuple[int, int]:
        j = int(math.floor((p[0] - self.origin[0]) / self.resolution + 0.5))
        i = int(math.floor((p[1] - self.origin[1]) / self.resolution + 0.5))
        return i, j

    def center_of(self, i: int, j: int) -> np.ndarray:
        return self.origin + self.resolution * np.array([j, i], dtype=np.float64)

    def in_bounds(self, i: int, j: int) -> bool:
        return 0 <= i < self.height and 0 <= j < self.width

    def navigable_cells(self) -> np.ndarray:
        return np.argwhere(self.navigable)

    def snap(self, points, radius: float = SNAP_RADIUS) -> np.ndarray:
        """_snap_to_navigable for many points: (m, 2) i32 cells, -1 rows when
        nothing navigable lies within radius (nav.py:103-119)."""
        self._check()
        pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 2))
        cells = np.empty((len(pts), 2), dtype=np.int32)
        nat.check(self.ctx.lib.nv_nav_snap(self.ctx.handle, nat.ptr(pts), len(pts),
                                           float(radius), nat.ptr(cells)))
        return cells


def _snap_to_navigable(grid: OccupancyGrid, p, radius: float = SNAP_RADIUS):
    c = grid.snap([p], radius)[0]
    return None if c[0] < 0 else (int(c[0]), int(c[1]))


def build_grid(ctx, bounds=None, resolution: float = DEFAULT_RESOLUTION,
               agent_radius: float = 0.1) -> OccupancyGrid:
    """Occupancy grid of the scene already uploaded to ``ctx``."""
    if resolution <= 0.0:
        raise NavError("resolution must be positive")
    if agent_radius < 0.0:
        raise NavError("agent_radius must be non-negative")
    b = None
    if bounds is not None:
        b = np.ascontiguousarray(np.asarray(bounds, dtype=np.float64).reshape(4))
        if not (b[2] > b[0] and b[3] > b[1]):
            raise ValueError("empty bounds")
    nx, ny = np.zeros(1, np.int64), np.zeros(1, np.int64)
    origin = np.zeros(2)
    nat.check(ctx.lib.nv_nav_build(ctx.handle, nat.ptr(b), float(resolution),
                                   float(agent_radius), nat.ptr(nx), nat.ptr(ny),
                                   nat.ptr(origin)))
    ctx._nav_gen = getattr(ctx, "_nav_gen", 0) + 1
    return OccupancyGrid(origin=origin, resolution=float(resolution), width=int(nx[0]),
                         height=int(ny[0]), ctx=ctx, gen=ctx._nav_gen)


def rasterize_navigable(segments, bounds, resolution: float = DEFAULT_RESOLUTION,
                        agent_radius: float = 0.1, device: int = 0) -> OccupancyGrid:
    """Cells whose centers clear every wall by agent_radius and lie inside the
    enclosure (nav.py:65-78 / geometry.navigable_mask)."""
    from .geometry import _upload_scene
    if resolution <= 0.0:
        raise NavError("resolution must be positive")
    if agent_radius < 0.0:
        raise NavError("agent_radius must be non-negative")
    segs = np.asarray(segments, dtype=np.float64).reshape(-1, 4)
    xmin, ymin, xmax, ymax = bounds
    if not (xmax > xmin and ymax > ymin):
        raise ValueError("empty bounds")
    ctx = nat.Context(device)
    n = len(segs)
    _upload_scene(ctx, segs, np.ones(n, np.uint16), np.full((n, 3), 0.5), 2.5,
                  (0.35, 0.33, 0.30), (0.85, 0.85, 0.85))
    return build_grid(ctx, bounds, resolution, agent_radius)


@dataclass(eq=False)
class DistanceField:
    """Geodesic distance to a fixed goal over an occupancy grid (nav.py:81-92)."""

    grid: OccupancyGrid
    goal: np.ndarray
    goal_cell: tuple[int, int]
    dist_device: object = field(repr=False)   # torch f64 (height, width) on the grid's GPU
    index: int = 0                            # field index inside dist_device's batch
    _host: dict = field(default_factory=dict, repr=False)

    @property
    def dist(self) -> np.ndarray:
        if "dist" not in self._host:
            self._host["dist"] = self.dist_device.cpu().numpy()
        return self._host["dist"]

    def interpolate(self, p) -> float:
        return geodesic_distance(self, p)


def distance_fields(grid: OccupancyGrid, goals):
    """Fields for many goals at once (one device relaxation over the batch):
    returns (fields tensor f64[k, h, w], goal cells (k, 2)).  Raises NavError
    when a goal has no navigable cell within SNAP_RADIUS."""
    import torch
    goals = np.asarray(goals, dtype=np.float64).reshape(-1, 2)
    cells = grid.snap(goals)
    bad = np.nonzero(cells[:, 0] < 0)[0]
    if len(bad):
        g = goals[bad[0]]
        raise NavError(f"goal ({g[0]:.3f}, {g[1]:.3f}) is not navigable")
    fields = torch.empty((len(goals), grid.height, grid.width), dtype=torch.float64,
                         device=f"cuda:{grid.ctx.device}")
    cc = np.ascontiguousarray(cells.astype(np.int32))
    nat.check(grid.ctx.lib.nv_nav_fields(grid.ctx.handle, nat.ptr(cc), len(cc), nat.ptr(fields),
                                         nat.stream_handle(f"cuda:{grid.ctx.device}")))
    return fields, cells


def distance_field(grid: OccupancyGrid, goal) -> DistanceField:
    """Dijkstra over 8-connected navigable cells from the goal (nav.py:122-132)."""
    fields, cells = distance_fields(grid, [goal])
    return DistanceField(grid=grid, goal=np.asarray(goal, dtype=np.float64),
                         goal_cell=(int(cells[0, 0]), int(cells[0, 1])), dist_device=fields[0])


def geodesic_distance(field: DistanceField, p) -> float:
    """Bilinear interpolation of the distance field at a world point (nav.py:135-166)."""
    import torch
    dev = field.dist_device.device
    pts = torch.tensor([[float(p[0]), float(p[1])]], dtype=torch.float64, device=dev)
    fid = torch.zeros(1, dtype=torch.int32, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    ctx = field.grid.ctx
    field.grid._check()
    nat.check(ctx.lib.nv_nav_geodesic(ctx.handle, nat.ptr(field.dist_device), nat.ptr(fid),
                                      nat.ptr(pts), 1, nat.ptr(out), nat.stream_handle(dev)))
    v = float(out.item())
    if math.isnan(v):
        raise NavError(f"point ({p[0]:.3f}, {p[1]:.3f}) outside grid bounds")
    return v


def sample_navigable(grid: OccupancyGrid, rng: np.random.Generator) -> np.ndarray:
    """Uniform over navigable cells, then uniform within the chosen cell (nav.py:169-177)."""
    cells = grid.navigable_cells()
    if len(cells) == 0:
        raise NavError("grid has no navigable space")
    i, j = cells[int(rng.integers(len(cells)))]
    center = grid.center_of(i, j)
    half = grid.resolution / 2.0
    return center + rng.uniform(-half, half, 2)
