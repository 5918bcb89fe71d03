"""The UNMODIFIED reference (navsim, installed into baseline/_ref from
/root/reference with pip --target) timed on this host's cores:

1. BASELINE.md section 3's methodology anchor: navsim.bench.run_benchmark on
   generate_scene(401) (acceptance criterion 11, tests/test_acceptance.py:
   328-339), rgbd at 128/256/512, 1 worker and all workers;
2. the reference's own Simulator.step (sim.py:202; render + raycast_grid +
   fill_frame + apply_forward) on the bench's C3 workload -- the same
   synthetic ~200k-triangle apartment, 256x256 RGB-D, seeded clearance-checked
   starts and uniform random actions -- with 1 worker and all workers, forked
   with the reference harness's Barrier + Queue pattern (bench.py:147-177),
   aggregate fps = sum(frames) / (max end - min start) (bench.py:170-174);
3. the repo's oracle port on the same sample (bench.cpu_baseline), so the
   port used as bench.py's reference arm is checked against the unmodified
   reference on the GPU box itself.

Prints one JSON object.  The GPU is not used.
"""
import json
import math
import multiprocessing as mp
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "navsim_numba"))

import numpy as np  # noqa: E402


def _scene_from_synth(cfg):
    from navsim.scene import Scene, WallSegment
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene(cfg)
    walls = [WallSegment(a=(float(s[0]), float(s[1])), b=(float(s[2]), float(s[3])),
                         semantic_id=int(k), albedo=tuple(float(v) for v in al))
             for s, k, al in zip(sc.segments, sc.semantic_ids, sc.albedo)]
    return sc, Scene(id=sc.name, walls=walls, floor_color=tuple(sc.floor_color),
                     ceiling_color=tuple(sc.ceiling_color), wall_height=sc.wall_height)


def _worker(graph, res, kinds, starts, acts, frames, warmup, barrier, queue, wid):
    from navsim.sensors import SensorConfig
    from navsim.sim import Action, AgentConfig, Simulator
    try:
        cfgs = tuple(SensorConfig(k, width=res, height=res) for k in kinds)
        sim = Simulator(graph, AgentConfig(), cfgs)
        x, y, h = starts[wid % len(starts)]
        sim.set_agent_state((x, y), h)
        amap = [Action.MOVE_FORWARD, Action.TURN_LEFT, Action.TURN_RIGHT]
        for k in range(warmup):
            sim.step(amap[int(acts[k % len(acts), wid % acts.shape[1]])])
        barrier.wait()
        t0 = time.perf_counter()
        for k in range(frames):
            sim.step(amap[int(acts[(warmup + k) % len(acts), wid % acts.shape[1]])])
        queue.put((wid, t0, time.perf_counter(), frames, ""))
    except Exception as e:  # report, never hang the coordinator
        try:
            barrier.wait(timeout=60)
        except Exception:
            pass
        queue.put((wid, 0.0, 0.0, 0, f"{type(e).__name__}: {e}"))


def _cell(graph, res, kinds, starts, acts, workers, frames, warmup):
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(workers + 1)
    queue = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(graph, res, kinds, starts, acts, frames, warmup,
                                               barrier, queue, w)) for w in range(workers)]
    for p in procs:
        p.start()
    barrier.wait()
    out = [queue.get() for _ in procs]
    for p in procs:
        p.join()
    errs = [r[4] for r in out if r[4]]
    if errs:
        return {"workers": workers, "error": "; ".join(errs)}
    wall = max(r[2] for r in out) - min(r[1] for r in out)
    return {"workers": workers, "fps_aggregate": sum(r[3] for r in out) / wall,
            "fps_per_worker": [r[3] / (r[2] - r[1]) for r in out], "frames_per_worker": frames}


def main():
    ncpu = os.cpu_count() or 1
    out = {"host_cpus": ncpu, "reference": REF, "cpu_model": None}
    try:
        with open("/proc/cpuinfo") as f:
            out["cpu_model"] = next(l.split(":", 1)[1].strip() for l in f
                                    if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    # 1. methodology anchor
    from navsim.bench import BenchConfig, run_benchmark
    from navsim.scene import build_scene_graph, generate_scene, save_scene
    t0 = time.time()
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "bench-scene.json")
        save_scene(generate_scene(401), path)
        rep = run_benchmark(BenchConfig(scene_path=path, resolutions=(128, 256, 512),
                                        sensor_sets=("rgbd",), worker_counts=(1, ncpu),
                                        frames=1200, warmup=200, repeats=1))
    out["anchor_generate_scene_401"] = {
        "cells": [{"sensors": c.sensors, "resolution": c.resolution, "workers": c.workers,
                   "fps_aggregate": c.fps_aggregate, "failed": c.failed} for c in rep.cells],
        "wall_s": time.time() - t0}
    # 2. the reference's Simulator.step on the C3 workload
    from paper_1904_01201_b200 import synth
    t0 = time.time()
    sc, scene = _scene_from_synth("C3")
    graph = build_scene_graph(scene)
    starts = synth.sample_poses(sc, 64, seed=1)
    acts = synth.random_actions(64, 4096, seed=2)
    out["c3_scene_build_s"] = time.time() - t0
    cells = []
    for workers, frames in ((1, 600), (ncpu, 400)):
        cells.append(_cell(graph, 256, ("rgb", "depth"), starts, acts, workers, frames, 200))
    out["c3_reference_simulator_step"] = {
        "workload": "C3 scene (99,820 segments), 256x256 RGB-D, seeded starts / uniform "
                    "random forward/left/right, warmup 200 frames per worker",
        "cells": cells}
    # 3. the oracle port on the same host (bench.py's reference arm)
    import bench
    out["oracle_port_c3"] = {"1_thread": bench.cpu_baseline("C3", seconds=10.0, threads=1),
                             "all_threads": bench.cpu_baseline("C3", seconds=10.0)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
