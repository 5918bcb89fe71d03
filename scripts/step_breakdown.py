"""Where the step time goes: per-step device time (one CUDA graph of K steps,
after a warm replay) of the bench workload under variants of the step.

  step_render      the bench's step (agent step + cast + fill)
  render_only      cast + fill at fixed poses (nv_render)
  step_only        the agent step alone (nv_step)
  forward_only     step_render with every action = forward (collisions, no sincos)
  turn_only        step_render with every action = turn (correctly rounded sincos)
  stop_only        step_render with every action = STOP (no kinematics)
usage: step_breakdown.py [CONFIG] [K]; prints one JSON object.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1904_01201_b200 import BatchSimulator, SensorConfig, synth  # noqa: E402


def timed(fn, K):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for k in range(K):
                fn(k)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3  # us per step


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    N, W, H, chans, key = bench.CONFIGS[cfg]
    sc = synth.config_scene(key)
    suite = tuple(SensorConfig(c, W, H) for c in chans) + (SensorConfig("gps_compass"),)
    sim = BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, N, sensor_configs=suite,
                         floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
    poses = synth.sample_poses(sc, N, seed=1)
    acts = torch.as_tensor(synth.random_actions(N, K + 8, seed=2), device="cuda:0")
    const = {a: torch.full((N,), a, dtype=torch.int8, device="cuda:0") for a in (0, 1, 3)}
    out = {"config": cfg, "envs": N, "steps": K, "us_per_step": {}}

    def run(name, fn):
        sim.reset(poses[:, :2], poses[:, 2])
        out["us_per_step"][name] = timed(fn, K)

    run("step_render", lambda k: sim.step(acts[k]))
    run("render_only", lambda k: sim.render())
    run("step_only", lambda k: sim.step(acts[k], render=False))
    run("forward_only", lambda k: sim.step(const[0]))
    run("turn_only", lambda k: sim.step(const[1]))
    run("stop_only", lambda k: sim.step(const[3]))
    run("step_only_forward", lambda k: sim.step(const[0], render=False))
    run("step_only_turn", lambda k: sim.step(const[1], render=False))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
