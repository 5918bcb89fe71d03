"""A few chained steps of every launch path at small sizes, for compute-sanitizer
(memcheck / racecheck / synccheck): thread-per-ray cast with per-env release,
warp-per-ray cast, the host-buffer step, the task step.  usage: compute-sanitizer
--tool memcheck python scripts/sanitize_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_01201_b200 import BatchSimulator, SensorConfig, synth  # noqa: E402
from paper_1904_01201_b200 import _native as nat  # noqa: E402

sc = synth.config_scene("C2")
for n, W, H, mode in ((80, 256, 64, nat.NV_CAST_THREAD), (8, 128, 32, nat.NV_CAST_WARP)):
    suite = (SensorConfig("rgb", W, H), SensorConfig("depth", W, H), SensorConfig("semantic", W, H),
             SensorConfig("gps_compass"))
    sim = BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
    nat.check(sim.ctx.lib.nv_set_cast_mode(sim.ctx.handle, mode))
    p = synth.sample_poses(sc, n, seed=3)
    sim.reset(p[:, :2], p[:, 2])
    acts = synth.random_actions(n, 4, seed=4)
    for s in range(4):
        sim.step(torch.as_tensor(acts[s], device="cuda:0"))
    out = {"gps": np.empty((n, 2)), "compass": np.empty(n), "collided": np.empty(n, np.uint8),
           "displacement": np.empty(n)}
    for s in range(3):
        sim.step_host(np.ascontiguousarray(acts[s]), out=out)
    torch.cuda.synchronize()
    print("ok", n, W, H, mode, float(sim.observations()["depth"].sum()))
