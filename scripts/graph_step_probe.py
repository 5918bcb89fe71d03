"""Per-step device time of the C3 step as (a) one CUDA graph of K steps and
(b) K back-to-back replays of a one-step graph (no host waits in between),
and (c) the host-buffer step loop (nv_step_render_host)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_01201_b200 import BatchSimulator, SensorConfig, synth  # noqa: E402

sc = synth.config_scene("C3")
N, K = 1024, 40
sim = BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, N,
                     sensor_configs=(SensorConfig("rgb", 256, 256), SensorConfig("depth", 256, 256)))
p = synth.sample_poses(sc, N, seed=1)
sim.reset(p[:, :2], p[:, 2])
acts = synth.random_actions(N, K + 10, seed=2)
da = torch.as_tensor(acts, device="cuda:0")
st = torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / K


with torch.cuda.stream(st):
    sim.step(da[0])
    torch.cuda.synchronize()
    gk = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gk, stream=st):
        for s in range(K):
            sim.step(da[s])
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1, stream=st):
        sim.step(da[0])
    gk.replay(); g1.replay()
    torch.cuda.synchronize()
    a = timed(lambda: gk.replay())
    b = timed(lambda: [g1.replay() for _ in range(K)])
out = {k: torch.empty(s, dtype=d).pin_memory() for k, s, d in
       (("gps", (N, 2), torch.float64), ("compass", (N,), torch.float64),
        ("collided", (N,), torch.uint8), ("displacement", (N,), torch.float64))}
host = torch.as_tensor(acts).pin_memory()
for s in range(5):
    sim.step_host(host[s].numpy(), out=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for s in range(K):
    sim.step_host(host[s].numpy(), out=out)
torch.cuda.synchronize()
c = (time.perf_counter() - t0) / K * 1e6
print(f"K-step graph {a:.1f} us/step; one-step graph x K {b:.1f} us/step; host-buffer step loop {c:.1f} us/step")
lib = sim.ctx.lib
if hasattr(lib, "nv_e2e_timing"):
    import ctypes
    buf = (ctypes.c_double * 3)()
    lib.nv_e2e_timing(buf)
    for s in range(K):
        sim.step_host(host[s].numpy(), out=out)
    torch.cuda.synchronize()
    lib.nv_e2e_timing(buf)
    n = buf[2] or 1
    print(f"host step: launches {buf[0]/n:.1f} us, spin {buf[1]/n:.1f} us per call")
    t0 = time.perf_counter()
    for s in range(K):
        t1 = time.perf_counter()
        sim.step_host(host[s].numpy(), out=out)
    torch.cuda.synchronize()
    print(f"python loop {(time.perf_counter() - t0) / K * 1e6:.1f} us/step")
