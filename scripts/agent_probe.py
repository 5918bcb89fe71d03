"""Agent-step time by action mix (C3, 1024 envs): all turns, all forward,
random -- CUDA events around the agent kernel (nv_profile)."""
import ctypes
import numpy as np
import torch
from paper_1904_01201_b200 import BatchSimulator, SensorConfig, synth
from paper_1904_01201_b200 import _native as nat

sc = synth.config_scene("C3")
N = 1024
suite = (SensorConfig("depth", 64, 16),)
sim = BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, N, sensor_configs=suite)
poses = synth.sample_poses(sc, N, seed=1)
sim.reset(poses[:, :2], poses[:, 2])
c = sim.ctx
for name, acts in (("turn", np.ones(N, np.int8)), ("forward", np.zeros(N, np.int8)),
                   ("random", synth.random_actions(N, 1, seed=3)[0])):
    a = torch.as_tensor(acts, device="cuda:0")
    for _ in range(3):
        sim.step(a, render=False)
    torch.cuda.synchronize()
    nat.check(c.lib.nv_profile(c.handle, 1))
    for _ in range(20):
        sim.step(a, render=False)
    torch.cuda.synchronize()
    ms = np.zeros(4)
    cnt = np.zeros(4, np.int64)
    nat.check(c.lib.nv_profile_read(c.handle, ms.ctypes.data_as(ctypes.c_void_p),
                                    cnt.ctypes.data_as(ctypes.c_void_p)))
    nat.check(c.lib.nv_profile(c.handle, 0))
    print(name, "agent_step us", round(ms[0] / max(cnt[0], 1) * 1e3, 2),
          "collided frac", float(sim.collided.float().mean()))
