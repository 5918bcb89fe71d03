"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front end of the nav/task oracle
(oracle/navsim_nav_oracle.c): occupancy rasterisation, distance fields,
geodesic queries, goal snapping and the PointGoal task step, restating
/root/reference/pkg/src/navsim/{geometry,nav,task}.py (file:line in the C
source).  Pinned against tests/golden/golden_task_*.npz by
tests/test_oracle_task_golden.py.  The product package never imports it.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import oracle as _o

_D = ctypes.c_double
_I64 = ctypes.c_int64
_P = ctypes.c_void_p
_ptr = _o._ptr

MAX_EPISODE_STEPS = 500   # task.py:24
SUCCESS_RADIUS = 0.2      # task.py:25
SNAP_RADIUS = 0.2         # nav.py:19


def _lib():
    lib = _o.lib()
    if not getattr(lib, "_nav_ready", False):
        lib.or_point_seg_dist.restype = _D
        lib.or_point_seg_dist.argtypes = [_P, _I64, _D, _D]
        lib.or_nav_dims.argtypes = [_D, _D, _D, _D, _D, _P, _P, _P, _P]
        lib.or_navigable_mask.argtypes = [_P, _I64, _D, _D, _D, _D, _D, _D, _P, _P]
        lib.or_dijkstra.argtypes = [_P, _I64, _I64, _I64, _I64, _D, _P]
        lib.or_snap.restype = ctypes.c_int
        lib.or_snap.argtypes = [_P, _I64, _I64, _D, _D, _D, _D, _D, _D, _P, _P]
        lib.or_geodesic.restype = _D
        lib.or_geodesic.argtypes = [_P, _I64, _I64, _D, _D, _D, _D, _D, _P]
        lib.or_spl.restype = _D
        lib.or_spl.argtypes = [ctypes.c_int, _D, _D]
        lib.or_reward.restype = _D
        lib.or_reward.argtypes = [_D, _D, ctypes.c_int, _D, _D]
        lib._nav_ready = True
    return lib


def bounds(segments):
    """Scene.bounds (scene.py:69-76)."""
    s = np.asarray(segments, dtype=np.float64).reshape(-1, 4)
    return (float(min(s[:, 0].min(), s[:, 2].min())), float(min(s[:, 1].min(), s[:, 3].min())),
            float(max(s[:, 0].max(), s[:, 2].max())), float(max(s[:, 1].max(), s[:, 3].max())))


class Grid:
    """OccupancyGrid (nav.py:27-62) built by navigable_mask."""

    def __init__(self, segments, bnds, resolution=0.05, agent_radius=0.1):
        segs = np.ascontiguousarray(np.asarray(segments, dtype=np.float64).reshape(-1, 4))
        L = _lib()
        nx, ny, ox, oy = _I64(), _I64(), _D(), _D()
        L.or_nav_dims(*[float(b) for b in bnds], float(resolution), ctypes.byref(nx),
                      ctypes.byref(ny), ctypes.byref(ox), ctypes.byref(oy))
        self.width, self.height = nx.value, ny.value
        self.origin = np.array([ox.value, oy.value])
        self.resolution = float(resolution)
        self.navigable = np.zeros((self.height, self.width), dtype=np.uint8)
        self.clearance = np.zeros((self.height, self.width))
        L.or_navigable_mask(_ptr(segs), len(segs), *[float(b) for b in bnds], float(resolution),
                            float(agent_radius), _ptr(self.navigable), _ptr(self.clearance))

    def cell_of(self, p):
        j = int(math.floor((p[0] - self.origin[0]) / self.resolution + 0.5))
        i = int(math.floor((p[1] - self.origin[1]) / self.resolution + 0.5))
        return i, j

    def center_of(self, i, j):
        return self.origin + self.resolution * np.array([j, i], dtype=np.float64)

    def snap(self, p, radius=SNAP_RADIUS):
        ci, cj = _I64(), _I64()
        ok = _lib().or_snap(_ptr(self.navigable), self.height, self.width, self.origin[0],
                            self.origin[1], self.resolution, float(p[0]), float(p[1]),
                            float(radius), ctypes.byref(ci), ctypes.byref(cj))
        return (ci.value, cj.value) if ok else None

    def field(self, goal_cell):
        d = np.empty((self.height, self.width))
        _lib().or_dijkstra(_ptr(self.navigable), self.height, self.width, int(goal_cell[0]),
                           int(goal_cell[1]), self.resolution, _ptr(d))
        return d

    def geodesic(self, dist, p):
        err = ctypes.c_int()
        v = _lib().or_geodesic(_ptr(np.ascontiguousarray(dist)), self.height, self.width,
                               self.origin[0], self.origin[1], self.resolution, float(p[0]),
                               float(p[1]), ctypes.byref(err))
        if err.value:
            raise ValueError("point outside grid bounds")
        return v


def spl(success, shortest, taken):
    return _lib().or_spl(int(bool(success)), float(shortest), float(taken))


def reward(d_prev, d_cur, reached, success_reward=10.0, step_penalty=-0.01):
    return _lib().or_reward(float(d_prev), float(d_cur), int(bool(reached)),
                            float(success_reward), float(step_penalty))


class TaskEnv:
    """Environment.reset/step (task.py:123-256) over the oracle simulator
    (oracle.OracleScene.step) -- task quantities only (no rendering)."""

    def __init__(self, scene: "_o.OracleScene", grid: Grid, radius=0.1, forward_step=0.25,
                 turn_angle=10.0, success_reward=10.0, step_penalty=-0.01):
        self.scene, self.grid = scene, grid
        self.radius, self.forward_step, self.turn_angle = radius, forward_step, turn_angle
        self.success_reward, self.step_penalty = success_reward, step_penalty

    def distance_to_goal(self, p):
        """Environment._distance_to_goal (task.py:160-177)."""
        goal = self.goal
        dx, dy = goal[0] - p[0], goal[1] - p[1]
        euclid = float(np.hypot(dx, dy))
        if euclid <= 1.0:
            if euclid < 1e-12:
                return 0.0
            t, _ = self.scene.raycast(p, np.array([[dx, dy]]))
            if not (t[0] <= 1.0):
                return euclid
        return self.grid.geodesic(self.field, p)

    def reset(self, start, heading, goal, gdsp):
        cell = self.grid.snap(goal)
        if cell is None:
            raise ValueError("goal not navigable")
        self.field = self.grid.field(cell)
        self.goal = np.asarray(goal, dtype=np.float64)
        start = np.asarray(start, dtype=np.float64)
        if self.scene.clearance(start) < self.radius:     # _snap_start (task.py:149-156)
            sc = self.grid.snap(start)
            if sc is None:
                raise ValueError("start not navigable")
            start = self.grid.center_of(*sc)
        self.state = [float(start[0]), float(start[1]), _o.wrap_angle(heading), 0.0, 0]
        self.gdsp = float(gdsp)
        self.steps = 0
        self.done = False
        self.d_last = self.distance_to_goal(start)
        return self.d_last

    def step(self, action: int):
        self.state, collided, moved = self.scene.step(self.state, action, self.radius,
                                                      self.forward_step, self.turn_angle)
        self.steps += 1
        d_prev, d_cur = self.d_last, self.distance_to_goal(self.state[:2])
        self.d_last = d_cur
        term, success = 0, False
        if action == 3:
            term, success = 1, d_cur <= SUCCESS_RADIUS
        elif self.steps >= MAX_EPISODE_STEPS:
            term = 2
        out = None
        if term:
            self.done = True
            out = dict(success=success, path_taken=self.state[3], steps=self.steps,
                       collisions=self.state[4], terminated_by=term,
                       spl=spl(success, self.gdsp, self.state[3]))
        r = reward(d_prev, d_cur, self.done and success, self.success_reward, self.step_penalty)
        return d_cur, r, self.done, collided, moved, out
