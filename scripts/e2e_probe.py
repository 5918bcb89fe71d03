"""Host-side cost of one end-to-end step (C3): wall time per step_host call
vs the device time per step, and the CUDA floor (replay + synchronize of a
one-kernel graph)."""
import time
import numpy as np
import torch
from paper_1904_01201_b200 import BatchSimulator, SensorConfig, synth

sc = synth.config_scene("C3")
N = 1024
sim = BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, N,
                     sensor_configs=(SensorConfig("rgb", 256, 256), SensorConfig("depth", 256, 256)))
p = synth.sample_poses(sc, N, seed=1)
sim.reset(p[:, :2], p[:, 2])
acts = synth.random_actions(N, 200, seed=2)
host = torch.as_tensor(acts).pin_memory()
out = {k: torch.empty(s, dtype=d).pin_memory() for k, s, d in
       (("gps", (N, 2), torch.float64), ("compass", (N,), torch.float64),
        ("collided", (N,), torch.uint8), ("displacement", (N,), torch.float64))}
for s in range(10):
    sim.step_host(host[s].numpy(), out=out)
torch.cuda.synchronize()
K = 150
t0 = time.perf_counter()
for s in range(K):
    sim.step_host(host[s % 200].numpy(), out=out)
wall = (time.perf_counter() - t0) / K * 1e6
# device time of the same step, back to back in one graph
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
da = torch.as_tensor(acts, device="cuda:0")
with torch.cuda.stream(st):
    sim.step(da[0])
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        for s in range(20):
            sim.step(da[s])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    g.replay()
e1.record()
torch.cuda.synchronize()
dev = e0.elapsed_time(e1) * 1e3 / 100
# CUDA floor: replay + synchronize of a tiny graph
x = torch.zeros(1, device="cuda:0")
g2 = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    with torch.cuda.graph(g2, stream=st):
        x.add_(1)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500):
    g2.replay()
    torch.cuda.current_stream().synchronize()
floor = (time.perf_counter() - t0) / 500 * 1e6
print(f"e2e wall per step {wall:.1f} us, device per step {dev:.1f} us, overhead {wall - dev:.1f} us; "
      f"tiny-graph replay+sync floor {floor:.1f} us")
# ctypes floor and the raw C call (no Python wrapper)
lib = sim.ctx.lib
t0 = time.perf_counter()
for _ in range(20000):
    lib.nv_version()
ct = (time.perf_counter() - t0) / 20000 * 1e6
args = sim._host_args
_, fn, h, cam, bits, tail, _ = args
a0 = host[0].numpy()
ptr = a0.ctypes.data
t0 = time.perf_counter()
for s in range(K):
    fn(h, ptr, cam, bits, *tail)
raw = (time.perf_counter() - t0) / K * 1e6
print(f"ctypes no-op call {ct:.2f} us; raw nv_step_render_host call {raw:.1f} us per step")
