"""PointGoal evaluation as BASELINE.json configs[4] names it, per GPU: C5 =
4096 envs over 8 GPUs -> 512 envs per GPU, 512x512 RGB-D, navmesh collision,
the ~1M-triangle scene (task.py:123-256, nav.py:117-166 on the device).

Times, on one GPU:
  * the navigation grid (clearance + navigable mask at 0.05 m) for the scene;
  * the goal distance fields (one Bellman-Ford field per distinct goal cell);
  * episode generation (geodesic distance of every start to every pooled goal);
  * BatchEnvironment.reset and the per-step cost of BatchEnvironment.step
    (agent step + task step + render, CUDA events) against the bare
    BatchSimulator step on the same envs;
  * a full evaluation: random forward/left/right until STOP at a fixed step,
    outcome records gathered (EpisodeOutcome, 40 B each) and summarised like
    agents.evaluate (agents.py:467-503).
Prints one JSON object.  usage: eval_pointgoal.py [CONFIG] [ENVS] [GOALS] [STEPS]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1904_01201_b200 import dist, nav, synth, task  # noqa: E402
from paper_1904_01201_b200.sensors import SensorConfig  # noqa: E402

RES = {"C3": 256, "C5": 512}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    n_goals = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    n_steps = int(sys.argv[4]) if len(sys.argv) > 4 else 200
    W = RES.get(cfg, 256)
    sc = synth.config_scene(cfg)
    out = {"config": cfg, "envs": N, "frame": f"{W}x{W} RGB-D", "segments": int(len(sc.segments)),
           "triangles": int(sc.n_triangles)}
    suite = (SensorConfig("rgb", W, W), SensorConfig("depth", W, W), SensorConfig("gps_compass"))
    # the navigation grid alone (its own context, like bench_nav.py): a
    # warm-up build, then a timed rebuild
    segs = sc.segments
    b = (float(min(segs[:, 0].min(), segs[:, 2].min())), float(min(segs[:, 1].min(), segs[:, 3].min())),
         float(max(segs[:, 0].max(), segs[:, 2].max())), float(max(segs[:, 1].max(), segs[:, 3].max())))
    g0 = nav.rasterize_navigable(segs, b)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g0 = nav.build_grid(g0.ctx, b)
    torch.cuda.synchronize()
    out["grid"] = {"nx": g0.width, "ny": g0.height, "cells": g0.width * g0.height,
                   "resolution_m": g0.resolution, "navigable": int(g0.navigable.sum()),
                   "build_s": time.perf_counter() - t0}
    del g0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    env = task.BatchEnvironment((sc.segments, sc.semantic_ids, sc.albedo), N, sensor_configs=suite,
                                max_steps=task.MAX_EPISODE_STEPS)
    torch.cuda.synchronize()
    out["env_build_s"] = time.perf_counter() - t0  # scene upload + navigation grid
    g = env.grid
    # episodes (geodesic distances to a pooled goal set, on device fields)
    shard = dist.EnvShard(N, 1, 0)
    t0 = time.perf_counter()
    eps = synth.pointgoal_episodes(env, sc, N, seed=11, n_goals=n_goals)
    torch.cuda.synchronize()
    out["episode_generation_s"] = time.perf_counter() - t0
    mask = np.array([e is not None for e in eps])
    out["episodes"] = int(mask.sum())
    dummy = next(e for e in eps if e is not None)
    # the same envs and starts stepped by the bare simulator (no task layer yet), K steps
    K = 20
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sacts = torch.as_tensor(synth.random_actions(N, K, seed=12), device=env.dev)
    sacts[sacts == 3] = 0
    env.sim.reset(np.stack([[e.start_position[0], e.start_position[1]] if e else
                            [dummy.start_position[0], dummy.start_position[1]] for e in eps]),
                  np.array([e.start_heading if e else dummy.start_heading for e in eps]))
    for t in range(3):
        env.sim.step(sacts[t])
    torch.cuda.synchronize()
    ev0.record()
    for t in range(K):
        env.sim.step(sacts[t])
    ev1.record()
    torch.cuda.synchronize()
    out["sim_ms_per_step"] = ev0.elapsed_time(ev1) / K
    t0 = time.perf_counter()
    env.reset([e if e is not None else dummy for e in eps], mask=mask)
    torch.cuda.synchronize()
    out["reset_s"] = time.perf_counter() - t0
    out["distinct_goal_fields"] = int(env.fields.shape[0])
    out["field_bytes"] = int(env.fields.numel() * 8)
    # fields alone: rebuild them for the distinct goal cells
    cells = np.asarray(list(env._field_of.keys()), dtype=np.int32)
    f = torch.empty((len(cells), g.height, g.width), dtype=torch.float64, device=env.dev)
    from paper_1904_01201_b200 import _native as nat
    c = env.sim.ctx
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nat.check(c.lib.nv_nav_fields(c.handle, nat.ptr(np.ascontiguousarray(cells)), len(cells),
                                  nat.ptr(f), nat.stream_handle(env.dev)))
    torch.cuda.synchronize()
    tf = time.perf_counter() - t0
    out["fields"] = {"count": int(len(cells)), "build_s": tf, "per_field_ms": tf / len(cells) * 1e3,
                     "bit_identical_to_reset_fields": bool(torch.equal(f, env.fields[:len(cells)]))}
    del f
    # per-step cost: task step + render vs the bare simulator step
    acts = torch.as_tensor(synth.random_actions(N, n_steps, seed=11), device=env.dev)
    acts[n_steps - 1] = 3
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for t in range(n_steps):
        env.step(acts[t])
    ev[1].record()
    torch.cuda.synchronize()
    t_eval = ev[0].elapsed_time(ev[1])
    done = env.done.clone() & torch.as_tensor(mask.astype(np.uint8), device=env.dev)
    t0 = time.perf_counter()
    rec = dist.gather_records(env.outcome.contiguous(), 1)
    summary = dist.outcome_summary(rec.cpu().numpy(), done.cpu().numpy())
    out["outcome_gather_s"] = time.perf_counter() - t0
    summary["policy"] = f"uniform random forward/left/right for {n_steps - 1} steps, then STOP"
    out["evaluation"] = summary
    out["eval_steps"] = n_steps
    out["eval_ms_per_step"] = t_eval / n_steps
    out["eval_frames_per_s"] = N * n_steps / (t_eval / 1e3)
    out["note"] = ("eval_ms_per_step includes envs already finished (frozen, re-rendered each "
                   "step) and the task arithmetic; per-GPU share of BASELINE configs[4] "
                   "(4096 envs over 8 GPUs)")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
