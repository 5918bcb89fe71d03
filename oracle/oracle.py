"""TEST INFRASTRUCTURE ONLY -- ctypes/numpy front end of the C oracle.

The oracle is a CPU restatement of the reference hot path (navsim,
/root/reference/pkg/src/navsim; see oracle/navsim_oracle.c for the per-function
file:line citations).  It is the parity checker for tests/, the thing
__graft_entry__.smoke() checks against, and the CPU baseline timed by
bench.py.  The product package (paper_1904_01201_b200) never imports it.

Pinning: tests/test_oracle_golden.py checks every function here bit-exactly
against tests/golden/*.npz, which tests/golden/make_golden.py produced by
running the unmodified reference (numba) in the build container.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libnavsim_oracle.so")

_D = ctypes.c_double
_I64 = ctypes.c_int64
_P = ctypes.c_void_p


def build() -> str:
    """Compile the oracle library (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def _load():
    if not os.path.exists(LIB_PATH):
        build()
    lib = ctypes.CDLL(LIB_PATH)
    lib.or_scene_create.restype = _P
    lib.or_scene_create.argtypes = [_P, _P, _P, _I64, _D, _P, _P]
    lib.or_scene_destroy.argtypes = [_P]
    lib.or_scene_grid.argtypes = [_P, _P, _P, _P, _P, _P]
    lib.or_scene_grid_copy.argtypes = [_P, _P, _P]
    lib.or_scene_raycast.argtypes = [_P, _D, _D, _P, _P, _I64, _D, ctypes.c_int, _P, _P]
    lib.or_cast_disc.argtypes = [_P, _D, _D, _D, _D, _D, _P, _P, _P, _P]
    lib.or_clearance.restype = _D
    lib.or_clearance.argtypes = [_P, _D, _D, _D]
    lib.or_wrap_angle.restype = _D
    lib.or_wrap_angle.argtypes = [_D]
    lib.or_step.restype = ctypes.c_int
    lib.or_step.argtypes = [_P, _P, _P, _P, _P, _P, ctypes.c_int, _D, _D, _D, _P]
    lib.or_render.argtypes = [_P, _D, _D, _D, _D, _I64, _I64, _D, _D, _D, ctypes.c_int,
                              _P, _P, _P]
    lib.or_fill_frame.argtypes = [_P, _P, _I64, _I64, _D, _D, _D, _D, _P, _P, _P, _P,
                                  _P, _P, _P, _P, _P, _P, _P]
    lib.or_column_directions.argtypes = [_D, _I64, _D, _P, _P]
    lib.or_gps_compass.argtypes = [_D, _D, _D, _D, _D, _D, _P, _P]
    lib.or_batch_step_render.argtypes = [_P, _I64, _P, _P, _P, _P, _P, _P, _D, _D, _D,
                                         _D, _I64, _I64, _D, _D, _P, _P, _P, ctypes.c_int,
                                         ctypes.c_int]
    lib.or_bench_cell.restype = _D
    lib.or_bench_cell.argtypes = [_P, _I64, _P, _P, _P, _P, _I64, _D, _D, _D, _D, _I64, _I64, _D,
                                  _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D,
                                  _P]
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def focal_of(width: int, hfov: float) -> float:
    """SensorConfig.focal, src/sensors.py:55-57."""
    return (width * 0.5) / math.tan(math.radians(hfov) * 0.5)


class OracleScene:
    """RenderGeometry + SegmentIndex restated (src/sensors.py:81-93,
    src/geometry.py:100-206)."""

    def __init__(self, segments, semantic_ids, albedo, wall_height=2.5,
                 floor_color=(0.35, 0.33, 0.30), ceiling_color=(0.85, 0.85, 0.85)):
        self.segments = np.ascontiguousarray(np.asarray(segments, dtype=np.float64).reshape(-1, 4))
        self.semantic_ids = np.ascontiguousarray(semantic_ids, dtype=np.uint16)
        self.albedo = np.ascontiguousarray(np.asarray(albedo, dtype=np.float64).reshape(-1, 3))
        self.wall_height = float(wall_height)
        self.floor_color = np.ascontiguousarray(floor_color, dtype=np.float64)
        self.ceiling_color = np.ascontiguousarray(ceiling_color, dtype=np.float64)
        self._h = lib().or_scene_create(_ptr(self.segments), _ptr(self.semantic_ids),
                                        _ptr(self.albedo), len(self.segments),
                                        self.wall_height, _ptr(self.floor_color),
                                        _ptr(self.ceiling_color))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_scene_destroy(self._h)
            self._h = None

    def grid(self):
        x0, y0 = ctypes.c_double(), ctypes.c_double()
        nx, ny, ni = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        lib().or_scene_grid(self._h, ctypes.byref(x0), ctypes.byref(y0), ctypes.byref(nx),
                            ctypes.byref(ny), ctypes.byref(ni))
        starts = np.empty(nx.value * ny.value + 1, dtype=np.int64)
        items = np.empty(ni.value, dtype=np.int64)
        lib().or_scene_grid_copy(self._h, _ptr(starts), _ptr(items))
        return x0.value, y0.value, nx.value, ny.value, starts, items

    def raycast(self, origin, dirs, t_max=1e9, brute=False):
        d = np.asarray(dirs, dtype=np.float64).reshape(-1, 2)
        dx = np.ascontiguousarray(d[:, 0])
        dy = np.ascontiguousarray(d[:, 1])
        t = np.empty(len(d))
        i = np.empty(len(d), dtype=np.int64)
        lib().or_scene_raycast(self._h, float(origin[0]), float(origin[1]), _ptr(dx), _ptr(dy),
                               len(d), float(t_max), int(brute), _ptr(t), _ptr(i))
        return t, i

    def cast_disc(self, pos, motion, radius):
        t, tx, ty = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        i = ctypes.c_int64()
        lib().or_cast_disc(self._h, float(pos[0]), float(pos[1]), float(motion[0]),
                           float(motion[1]), float(radius), ctypes.byref(t), ctypes.byref(i),
                           ctypes.byref(tx), ctypes.byref(ty))
        return t.value, i.value, np.array([tx.value, ty.value])

    def clearance(self, pos, search_radius=2.0):
        return lib().or_clearance(self._h, float(pos[0]), float(pos[1]), float(search_radius))

    def render(self, position, heading, sensor_height, width=256, height=256, hfov=90.0,
               max_range=10.0, want=("rgb", "depth", "semantic"), t_max=1e9, brute=False,
               focal=None):
        """sensors.render for one (w, h, hfov, max_range) group."""
        f = focal_of(width, hfov) if focal is None else focal
        depth = np.empty((height, width)) if "depth" in want else None
        rgb = np.empty((height, width, 3)) if "rgb" in want else None
        sem = np.empty((height, width), dtype=np.uint16) if "semantic" in want else None
        lib().or_render(self._h, float(position[0]), float(position[1]), float(heading),
                        float(sensor_height), width, height, f, float(max_range), float(t_max),
                        int(brute), _ptr(depth), _ptr(rgb), _ptr(sem))
        return rgb, depth, sem

    def step(self, state, action: int, radius=0.1, forward_step=0.25, turn_angle=10.0):
        """Simulator.step kinematics (src/sim.py:202-219); state = [x, y, h, path, coll]."""
        x, y, h, pl = (ctypes.c_double(float(v)) for v in state[:4])
        c = ctypes.c_int64(int(state[4]))
        moved = ctypes.c_double()
        collided = lib().or_step(self._h, ctypes.byref(x), ctypes.byref(y), ctypes.byref(h),
                                 ctypes.byref(pl), ctypes.byref(c), int(action), float(radius),
                                 float(forward_step), math.radians(turn_angle),
                                 ctypes.byref(moved))
        return [x.value, y.value, h.value, pl.value, c.value], bool(collided), moved.value

    def batch_step_render(self, x, y, h, path, coll, actions, radius, forward_step,
                          turn_angle, sensor_height, width, height, focal, max_range,
                          depth, rgb, sem, nthreads, per_thread_frames=False):
        """CPU baseline: N envs step + render, nthreads workers; frames one
        per env, or (per_thread_frames) one per worker thread, reused."""
        lib().or_batch_step_render(self._h, len(x), _ptr(x), _ptr(y), _ptr(h), _ptr(path),
                                   _ptr(coll), _ptr(actions), radius, forward_step,
                                   math.radians(turn_angle), sensor_height, width, height,
                                   focal, max_range, _ptr(depth), _ptr(rgb), _ptr(sem),
                                   int(nthreads), int(bool(per_thread_frames)))


def bench_cell(scene: "OracleScene", poses, actions, width, height, focal, channels, threads,
               seconds, radius=0.1, forward_step=0.25, turn_angle=10.0, sensor_height=1.5,
               max_range=10.0):
    """The reference harness's cell (src/bench.py:128-177) on the C port:
    ``threads`` workers, one env each (start pose poses[w % N], actions
    column w % N of the (steps, N) table, cycled), Simulator.step + render
    for ``seconds``; returns (aggregate frames/s = sum(frames) / (max end -
    min start), frames)."""
    poses = np.ascontiguousarray(np.asarray(poses, dtype=np.float64))
    acts = np.ascontiguousarray(np.asarray(actions, dtype=np.int8))
    x0, y0, h0 = (np.ascontiguousarray(poses[:, k]) for k in range(3))
    frames = np.zeros(1, dtype=np.int64)
    fps = lib().or_bench_cell(scene._h, len(poses), _ptr(x0), _ptr(y0), _ptr(h0), _ptr(acts),
                              acts.shape[0], radius, forward_step, math.radians(turn_angle),
                              sensor_height, width, height, focal, max_range,
                              int("rgb" in channels), int("depth" in channels),
                              int("semantic" in channels), int(threads), float(seconds),
                              _ptr(frames))
    return fps, int(frames[0])


def wrap_angle(theta: float) -> float:
    return lib().or_wrap_angle(float(theta))


def column_directions(heading, width, focal):
    dx = np.empty(width)
    dy = np.empty(width)
    lib().or_column_directions(float(heading), width, float(focal), _ptr(dx), _ptr(dy))
    return dx, dy


def gps_compass(x, y, h, ox, oy, oh):
    g = np.empty(2)
    c = ctypes.c_double()
    lib().or_gps_compass(x, y, h, ox, oy, oh, _ptr(g), ctypes.byref(c))
    return g, c.value


def fill_frame(t_col, i_col, height, width, focal, cam_h, wall_h, max_range, albedo, sem_ids,
               nx, ny, dirx, diry, floor_color, ceil_color, want=("rgb", "depth", "semantic")):
    depth = np.empty((height, width)) if "depth" in want else None
    rgb = np.empty((height, width, 3)) if "rgb" in want else None
    sem = np.empty((height, width), dtype=np.uint16) if "semantic" in want else None
    args = [np.ascontiguousarray(a, dtype=dt) for a, dt in (
        (t_col, np.float64), (i_col, np.int64), (albedo, np.float64), (sem_ids, np.uint16),
        (nx, np.float64), (ny, np.float64), (dirx, np.float64), (diry, np.float64),
        (floor_color, np.float64), (ceil_color, np.float64))]
    lib().or_fill_frame(_ptr(args[0]), _ptr(args[1]), height, width, focal, cam_h, wall_h,
                        max_range, _ptr(args[2]), _ptr(args[3]), _ptr(args[4]), _ptr(args[5]),
                        _ptr(args[6]), _ptr(args[7]), _ptr(args[8]), _ptr(args[9]),
                        _ptr(depth), _ptr(rgb), _ptr(sem))
    return rgb, depth, sem
