"""The single-env drop-in ``Simulator`` (the API the reference's own callers
use: task.py:136, bench workers) against the reference's in-process
``Simulator.step`` (sim.py:202), same scene, same actions, 256x256 RGB-D,
one agent, one host thread, observations returned as the reference's host
arrays (rgb f64 [0,1], depth f64, gps/compass).

Rows: this repo's Simulator (GPU, C ABI) and -- when baseline/_ref holds the
unmodified reference (pip --target install) -- the reference Simulator.
Scenes: C1 (1-room, 1000 segments) and C3 (the ~200k-triangle apartment).
Prints one JSON object.
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "navsim_numba"))


def _scene(mod, sc):
    walls = [mod.WallSegment(a=(float(s[0]), float(s[1])), b=(float(s[2]), float(s[3])),
                             semantic_id=int(k), albedo=tuple(float(v) for v in al))
             for s, k, al in zip(sc.segments, sc.semantic_ids, sc.albedo)]
    return mod.build_scene_graph(mod.Scene(id=sc.name, walls=walls,
                                           floor_color=tuple(sc.floor_color),
                                           ceiling_color=tuple(sc.ceiling_color),
                                           wall_height=sc.wall_height))


def _time(sim_mod, scene_mod, sens_mod, sc, start, acts, warmup, steps):
    graph = _scene(scene_mod, sc)
    cfgs = (sens_mod.SensorConfig("rgb", 256, 256), sens_mod.SensorConfig("depth", 256, 256),
            sens_mod.SensorConfig("gps_compass"))
    sim = sim_mod.Simulator(graph, sim_mod.AgentConfig(), cfgs)
    sim.set_agent_state((float(start[0]), float(start[1])), float(start[2]))
    amap = [sim_mod.Action.MOVE_FORWARD, sim_mod.Action.TURN_LEFT, sim_mod.Action.TURN_RIGHT]
    for k in range(warmup):
        sim.step(amap[int(acts[k])])
    t0 = time.perf_counter()
    for k in range(steps):
        res, obs = sim.step(amap[int(acts[warmup + k])])
    dt = time.perf_counter() - t0
    return {"frames_per_s": steps / dt, "ms_per_step": dt / steps * 1e3, "steps": steps,
            "final_position": [float(v) for v in res.new_state.position],
            "final_heading": float(res.new_state.heading)}


def main():
    from paper_1904_01201_b200 import scene as our_scene
    from paper_1904_01201_b200 import sensors as our_sens
    from paper_1904_01201_b200 import sim as our_sim
    from paper_1904_01201_b200 import synth
    have_ref = os.path.isdir(os.path.join(REF, "navsim"))
    if have_ref:
        sys.path.insert(0, REF)
        from navsim import scene as ref_scene
        from navsim import sensors as ref_sens
        from navsim import sim as ref_sim
    out = {"frame": "256x256 RGB-D + gps_compass, one agent, one host thread", "rows": {}}
    for cfg in ("C1", "C3"):
        sc = synth.config_scene(cfg)
        start = synth.sample_poses(sc, 1, seed=3)[0]
        acts = synth.random_actions(1, 1200, seed=4)[:, 0]
        row = {"segments": int(len(sc.segments)),
               "repo_simulator": _time(our_sim, our_scene, our_sens, sc, start, acts, 50, 400)}
        if have_ref:
            row["reference_simulator"] = _time(ref_sim, ref_scene, ref_sens, sc, start, acts,
                                               50, 400)
            ro, rr = row["repo_simulator"], row["reference_simulator"]
            row["speedup"] = ro["frames_per_s"] / rr["frames_per_s"]
        out["rows"][cfg] = row
    print(json.dumps(out))


if __name__ == "__main__":
    main()
