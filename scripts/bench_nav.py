"""Measurement of the nav/task row on one GPU.

* occupancy grid (clearance + mask) and distance-field build on the device
  for the C3 apartment (100k segments, 0.05 m grid), wall-clock around the
  synchronous C ABI calls; per-field time for a batch of goals;
* the same on the CPU oracle (single thread) on a bounded sample: clearance
  rows extrapolated, one full Dijkstra field (the reference's algorithm);
* the task layer's per-step cost: BatchEnvironment.step vs the bare
  BatchSimulator step at 1024 envs x 256x256 RGB-D (CUDA events).
Prints one JSON object.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1904_01201_b200 import nav, synth, task  # noqa: E402
from paper_1904_01201_b200.sensors import SensorConfig  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    n_goals = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    sc = synth.config_scene(cfg)
    segs = sc.segments
    b = (float(min(segs[:, 0].min(), segs[:, 2].min())), float(min(segs[:, 1].min(), segs[:, 3].min())),
         float(max(segs[:, 0].max(), segs[:, 2].max())), float(max(segs[:, 1].max(), segs[:, 3].max())))
    out = {"scene": cfg, "segments": int(len(segs))}
    g = nav.rasterize_navigable(segs, b)        # warm-up (context, module load)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = nav.build_grid(g.ctx, b)
    t_grid = time.perf_counter() - t0
    cells = np.argwhere(g.navigable)
    out.update(grid={"nx": g.width, "ny": g.height, "cells": g.width * g.height,
                     "navigable": int(len(cells)), "build_s": t_grid})
    rng = np.random.default_rng(5)
    goals = [g.center_of(*cells[int(rng.integers(len(cells)))]) for _ in range(n_goals)]
    nav.distance_fields(g, goals[:1])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fields, fc = nav.distance_fields(g, goals)
    torch.cuda.synchronize()
    t_f = time.perf_counter() - t0
    out["fields"] = {"goals": n_goals, "build_s": t_f, "per_field_ms": t_f / n_goals * 1e3}
    # CPU oracle (single thread): one Dijkstra field on the same grid, and
    # clearance for a bounded band of rows (extrapolated)
    from oracle import nav_oracle as no
    import ctypes
    L = no._lib()
    mask = np.ascontiguousarray(g.navigable.astype(np.uint8))
    d = np.empty(mask.shape)
    t0 = time.perf_counter()
    L.or_dijkstra(mask.ctypes.data_as(ctypes.c_void_p), g.height, g.width, int(fc[0, 0]),
                  int(fc[0, 1]), g.resolution, d.ctypes.data_as(ctypes.c_void_p))
    t_dij = time.perf_counter() - t0
    same = bool(np.array_equal(d, fields[0].cpu().numpy()))
    sseg = np.ascontiguousarray(segs)
    rows = 2
    t0 = time.perf_counter()
    for i in range(rows):
        y = g.origin[1] + g.resolution * (g.height // 2 + i)
        for j in range(0, g.width, 8):
            L.or_point_seg_dist(sseg.ctypes.data_as(ctypes.c_void_p), len(sseg),
                                g.origin[0] + g.resolution * j, y)
    t_rows = time.perf_counter() - t0
    per_cell = t_rows / (rows * len(range(0, g.width, 8)))
    out["cpu_oracle"] = {"cores": 1, "dijkstra_field_s": t_dij, "field_bit_identical": same,
                         "clearance_per_cell_s": per_cell,
                         "clearance_grid_s_extrapolated": per_cell * g.width * g.height,
                         "sample": f"1 field; {rows} rows x every 8th cell of clearance"}
    # task layer per-step cost
    N, W = 1024, 256
    suite = (SensorConfig("rgb", W, W), SensorConfig("depth", W, W))
    env = task.BatchEnvironment((segs, sc.semantic_ids, sc.albedo), N, sensor_configs=suite)
    poses = synth.sample_poses(sc, N, seed=2)
    pool = synth.sample_poses(sc, 16 * N, seed=3)[:, :2]
    eps = []
    for k in range(N):
        s = poses[k, :2]
        dd = np.hypot(pool[:, 0] - s[0], pool[:, 1] - s[1])
        gl = pool[int(np.nonzero((dd >= 2.0) & (dd <= 10.0))[0][0])]
        eu = float(np.hypot(*(gl - s)))
        gd = eu  # stand-in shortest path (only SPL's scale depends on it)
        eps.append(task.Episode(f"e{k}", "x", tuple(s), float(poses[k, 2]), tuple(gl), gd, eu,
                                gd / eu if eu > 0 else 0.0))
    t0 = time.perf_counter()
    env.reset(eps)
    torch.cuda.synchronize()
    t_reset = time.perf_counter() - t0
    acts = torch.as_tensor(synth.random_actions(N, 40, seed=4), device="cuda:0")
    for s in range(5):
        env.step(acts[s])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    K = 30
    torch.cuda.synchronize()
    ev[0].record()
    for s in range(K):
        env.step(acts[5 + s])
    ev[1].record()
    for s in range(K):
        env.sim.step(acts[5 + s])
    ev[2].record()
    torch.cuda.synchronize()
    t_task = ev[0].elapsed_time(ev[1]) / K
    t_sim = ev[1].elapsed_time(ev[2]) / K
    out["task_step"] = {"envs": N, "frame": f"{W}x{W} RGB-D", "ms_per_step_with_task": t_task,
                        "ms_per_step_sim_only": t_sim, "task_overhead_ms": t_task - t_sim,
                        "reset_s": t_reset, "distinct_goal_fields": int(env.fields.shape[0])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
