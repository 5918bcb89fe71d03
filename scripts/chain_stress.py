"""Stress the chained step at small batches (writer grids smaller than the
GPU): R repetitions of S back-to-back steps against serialised launches, per
config; prints the number of mismatching repetitions and handshake faults.
usage: chain_stress.py [R]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1904_01201_b200 as nb  # noqa: E402
from paper_1904_01201_b200 import _native as nat, synth  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 10
CASES = (("C2", 128, 128, 3, 60, 1), ("C1", 256, 256, 1, 60, 1),
         ("C2", 128, 128, 16, 60, 0), ("C1", 256, 256, 1, 60, 0),
         # full writer grids with thread-per-ray casts (release, pose records)
         ("C3", 256, 256, 256, 30, 0), ("C2", 256, 128, 160, 30, 0),
         ("C3", 256, 256, 1024, 20, 0))
only = sys.argv[2] if len(sys.argv) > 2 else None
for cfg, W, H, n, steps, mode in CASES:
    if only == "full" and n < 100:
        continue
    sc = synth.config_scene(cfg)
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("gps_compass"))
    bad = faults = 0
    for r in range(R):
        sims = []
        for overlap in (0, 1):
            sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
            nat.check(sim.ctx.lib.nv_set_overlap(sim.ctx.handle, overlap))
            nat.check(sim.ctx.lib.nv_set_cast_mode(sim.ctx.handle, mode))
            poses = synth.sample_poses(sc, n, seed=100 + r)
            sim.reset(poses[:, :2], poses[:, 2])
            sims.append(sim)
        acts = torch.as_tensor(synth.random_actions(n, steps, seed=200 + r), device="cuda:0")
        s0, s1 = sims
        for s in range(steps):
            s1.step(acts[s])
        for s in range(steps):
            s0.step(acts[s])
            torch.cuda.synchronize()
        torch.cuda.synchronize()
        faults += s1.ctx.faults() != 0
        o0, o1 = s0.observations(), s1.observations()
        same = all(torch.equal(o0[k], o1[k]) for k in ("rgb", "depth", "gps", "compass"))
        same &= all(torch.equal(a, b) for a, b in zip(s0.state(), s1.state()))
        bad += not same
    print(f"{cfg} n={n} mode={mode}: {bad}/{R} mismatching runs, {faults} with faults")
