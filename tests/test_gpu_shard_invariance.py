"""Sharding invariance ("seeds compose", src/seeding.py:13-23):
per-env results do not depend on how many ranks the envs are spread over.

Two ranks on one GPU (spawned processes, gloo for the collective) each own
half of an 11-env batch (uneven split, non-zero env_offset on rank 1) and are
compared bit for bit with a single-rank run of the same 11 envs: every frame
of every step (RGB, depth with inverse-depth noise ON, semantic), poses, step
results, and the all-gathered 40-byte EpisodeOutcome records of a PointGoal
evaluation (the path's one collective).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N_TOTAL = 11
STEPS = 8
SIGMA = 0.3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_run(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1904_01201_b200 import BatchSimulator, SensorConfig, synth, task
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200.dist import EnvShard, pointgoal_eval
    shard = EnvShard(n_total=N_TOTAL, world=world, rank=rank)
    sc = synth.config_scene("C2")
    W, H = 128, 64
    suite = (SensorConfig("rgb", W, H), SensorConfig("depth", W, H), SensorConfig("semantic", W, H),
             SensorConfig("gps_compass"))
    sim = BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, shard.n_local,
                         sensor_configs=suite, floor_color=sc.floor_color,
                         ceiling_color=sc.ceiling_color)
    nat.check(sim.ctx.lib.nv_depth_noise(sim.ctx.handle, SIGMA, 77, shard.lo))
    poses = synth.sample_poses(sc, shard.n_local, seed=3, first=shard.lo)
    sim.reset(poses[:, :2], poses[:, 2])
    acts = synth.random_actions(N_TOTAL, STEPS, seed=4)[:, shard.lo:shard.hi]
    out = {k: [] for k in ("rgb", "depth", "semantic", "gps", "compass", "collided", "disp", "xy",
                           "h")}
    for t in range(STEPS):
        sim.step(torch.as_tensor(np.ascontiguousarray(acts[t]), device="cuda:0"))
        torch.cuda.synchronize()
        o = sim.observations()
        for k in ("rgb", "depth", "gps", "compass"):
            out[k].append(o[k].cpu().numpy())
        out["semantic"].append(o["semantic"].view(torch.int16).cpu().numpy())
        out["collided"].append(sim.collided.cpu().numpy())
        out["disp"].append(sim.displacement.cpu().numpy())
        xy, h, _, _ = sim.state()
        out["xy"].append(xy.cpu().numpy())
        out["h"].append(h.cpu().numpy())
    env = task.BatchEnvironment((sc.segments, sc.semantic_ids, sc.albedo), shard.n_local,
                                sensor_configs=(SensorConfig("depth", 64, 16),), max_steps=500,
                                depth_noise_sigma=SIGMA, noise_seed=5, env_offset=shard.lo)
    summary, rec, fin = pointgoal_eval(env, sc, shard, world, n_steps=24, seed=13)
    res = {k: np.stack(v, axis=1) for k, v in out.items()}  # env-major
    res["records"] = rec.cpu().numpy()
    res["finished"] = fin.cpu().numpy()
    res["episodes"] = np.array([summary["episodes"]])
    np.savez(out_path, **res)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _spawn(world, tmp_path):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    paths = [str(tmp_path / f"w{world}_r{r}.npz") for r in range(world)]
    procs = [ctx.Process(target=_shard_run, args=(r, world, port, paths[r])) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    return [dict(np.load(p)) for p in paths]


def test_two_ranks_match_one_rank(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    one = _spawn(1, tmp_path)[0]
    two = _spawn(2, tmp_path)
    for k in ("rgb", "depth", "semantic", "gps", "compass", "collided", "disp", "xy", "h"):
        cat = np.concatenate([two[0][k], two[1][k]], axis=0)
        assert cat.shape == one[k].shape, k
        assert np.array_equal(cat.view(np.uint8), one[k].view(np.uint8)), k
    # the noise is on (not a vacuous check): without it the bottom (floor) row
    # has one depth; with it every pixel draws its own
    assert len(np.unique(one["depth"][0, 0, -1])) > 16
    # the gathered EpisodeOutcome records: same bytes on every rank, same as one rank
    assert int(one["episodes"][0]) > 0
    for r in range(2):
        assert np.array_equal(two[r]["records"], one["records"])
        assert np.array_equal(two[r]["finished"], one["finished"])
