"""Study build (NV_STUDY_WAITSTAT=1): how long the release writer's loader
waits for each item's env to be cast, per item rank, over K C3 steps in a
CUDA graph.  usage: NAVSIM_B200_LIB=<study .so> waitstat_probe.py [CONFIG] [K]"""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1904_01201_b200 import BatchSimulator, SensorConfig, synth  # noqa: E402
from paper_1904_01201_b200 import _native as nat  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    N, W, H, chans, key = bench.CONFIGS[cfg]
    sc = synth.config_scene(key)
    suite = tuple(SensorConfig(c, W, H) for c in chans) + (SensorConfig("gps_compass"),)
    sim = BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, N, sensor_configs=suite,
                         floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
    poses = synth.sample_poses(sc, N, seed=1)
    sim.reset(poses[:, :2], poses[:, 2])
    acts = torch.as_tensor(synth.random_actions(N, K + 8, seed=2), device="cuda:0")
    lib = nat.load()
    fn = lib.nv_study_waitstat
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p]
    buf = (ctypes.c_ulonglong * 16)()
    for s in range(5):
        sim.step(acts[s])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for k in range(K):
                sim.step(acts[k])
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    fn(buf)
    g.replay()
    torch.cuda.synchronize()
    fn(buf)
    ns = list(buf)
    out = {"config": cfg, "steps": K,
           "wait_us_per_step_by_item_rank": [round(ns[i] / 1e3 / K, 2) for i in range(8)],
           "items_per_step_by_rank": [ns[8 + i] / K for i in range(8)],
           "mean_wait_us_per_item_by_rank": [round(ns[i] / max(1, ns[8 + i]) / 1e3, 3) for i in range(8)]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
