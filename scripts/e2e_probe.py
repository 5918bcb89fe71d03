"""Host-side timeline of the host-buffer step (nv_step_render_host) at a
bench config: per call, the time spent inside the C call (launch + wait for
the casts) and outside it (Python), and the steady-state period.
usage: e2e_probe.py [CONFIG] [K]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1904_01201_b200 import BatchSimulator, SensorConfig, synth  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    N, W, H, chans, key = bench.CONFIGS[cfg]
    sc = synth.config_scene(key)
    suite = tuple(SensorConfig(c, W, H) for c in chans) + (SensorConfig("gps_compass"),)
    sim = BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, N, sensor_configs=suite,
                         floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
    poses = synth.sample_poses(sc, N, seed=1)
    sim.reset(poses[:, :2], poses[:, 2])
    acts = torch.as_tensor(synth.random_actions(N, K + 8, seed=2)).pin_memory()
    out = {"gps": torch.empty((N, 2), dtype=torch.float64).pin_memory(),
           "compass": torch.empty((N,), dtype=torch.float64).pin_memory(),
           "collided": torch.empty((N,), dtype=torch.uint8).pin_memory(),
           "displacement": torch.empty((N,), dtype=torch.float64).pin_memory()}
    a_np = [acts[s].numpy() for s in range(K + 8)]
    for s in range(5):
        sim.step_host(a_np[s], out=out)
    torch.cuda.synchronize()
    t_in = np.zeros(K)
    t_start = np.zeros(K)
    for s in range(K):
        t0 = time.perf_counter()
        sim.step_host(a_np[s + 5], out=out)
        t1 = time.perf_counter()
        t_start[s] = t0
        t_in[s] = t1 - t0
    torch.cuda.synchronize()
    t_end = time.perf_counter()
    period = np.diff(t_start) * 1e6
    res = {"config": cfg, "steps": K,
           "period_us": {"median": float(np.median(period)), "p10": float(np.percentile(period, 10)),
                         "p90": float(np.percentile(period, 90))},
           "in_call_us_median": float(np.median(t_in) * 1e6),
           "outside_call_us_median": float(np.median(period - t_in[:-1] * 1e6)),
           "total_per_step_us": (t_end - t_start[0]) / K * 1e6}
    print(json.dumps(res))


if __name__ == "__main__":
    main()


def short_runs(cfg="C3", K=20, reps=5):
    """Per-call host times of K-step runs started from an idle GPU (the
    bench's e2e protocol): where the fixed per-run cost goes."""
    N, W, H, chans, key = bench.CONFIGS[cfg]
    sc = synth.config_scene(key)
    suite = tuple(SensorConfig(c, W, H) for c in chans) + (SensorConfig("gps_compass"),)
    sim = BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, N, sensor_configs=suite,
                         floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
    poses = synth.sample_poses(sc, N, seed=1)
    sim.reset(poses[:, :2], poses[:, 2])
    acts = torch.as_tensor(synth.random_actions(N, K * reps + 8, seed=2)).pin_memory()
    out = {"gps": torch.empty((N, 2), dtype=torch.float64).pin_memory(),
           "compass": torch.empty((N,), dtype=torch.float64).pin_memory(),
           "collided": torch.empty((N,), dtype=torch.uint8).pin_memory(),
           "displacement": torch.empty((N,), dtype=torch.float64).pin_memory()}
    a_np = [acts[s].numpy() for s in range(K * reps + 8)]
    for s in range(3):
        sim.step_host(a_np[s], out=out)
    rows = []
    for r in range(reps):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        for s in range(K):
            sim.step_host(a_np[3 + r * K + s], out=out)
            t.append(time.perf_counter())
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        d = np.diff(t) * 1e6
        rows.append({"calls_us": [round(x, 1) for x in d[:-1]], "final_sync_us": round(d[-1], 1),
                     "total_us": round((t[-1] - t[0]) * 1e6, 1)})
    print(json.dumps({"config": cfg, "K": K, "runs": rows}))


if __name__ == "__main__" and os.environ.get("E2E_SHORT"):
    short_runs()
