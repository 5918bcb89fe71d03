"""Cast event counts per ray (study build: NV_CAST_STATS=1, load it with
NAVSIM_B200_LIB): cells, non-empty cells, run boxes tested/passed, f32 side
tests, exact tests and why they fail -- C3, 1024 envs x 256 columns."""
import ctypes
import numpy as np
import torch
from paper_1904_01201_b200 import BatchSimulator, SensorConfig, synth

sc = synth.config_scene("C3")
N = 1024
sim = BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, N,
                     sensor_configs=(SensorConfig("rgb", 256, 256), SensorConfig("depth", 256, 256)))
poses = synth.sample_poses(sc, N, seed=1)
sim.reset(poses[:, :2], poses[:, 2])
c = sim.ctx
acts = synth.random_actions(N, 12, seed=2)
st = np.zeros(16, np.uint64)
rd = c.lib.nv_cast_stats_read
rd.argtypes = [ctypes.c_void_p, ctypes.c_int]
for s in range(2):
    sim.step(torch.as_tensor(acts[s], device="cuda:0"))
rd(st.ctypes.data, 1)
steps = 10
for s in range(2, 2 + steps):
    sim.step(torch.as_tensor(acts[s], device="cuda:0"))
torch.cuda.synchronize()
rd(st.ctypes.data, 0)
rays = N * 256 * steps
names = ["cells visited", "non-empty cells", "run boxes tested", "entries side-tested (f32)",
         "side-test survivors (exact pre)", "seg_pre pass (div)", "run boxes passed",
         "pass but t<0", "pre-reject: behind", "pre-reject: beyond best", "pre-reject: r/den"]
for k, n in enumerate(names):
    print(f"{n:34s} {st[k] / rays:8.2f} per ray")
