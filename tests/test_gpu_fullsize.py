"""Parity at BASELINE.json's full sizes, the bench's own workloads and default
paths (warp-specialised writer, thread-per-ray DDA):

* C3: 1024 envs x 256x256 RGB-D(-S) on the ~200k-triangle apartment;
* C5: 512 envs (4096 over 8 GPUs) x 512x512 RGB-D(-S) on the ~1M-triangle
  scene (~500k segments, 161x155 grid; two warp segments per frame row in
  the writer, row-banded work items), plus a small C5 batch compared with
  the oracle in every env at every step;

* a seeded sample of envs against the oracle at every step (poses 1e-6,
  semantic/coverage exact, depth 1e-5 rel, RGB 1/255);
* size-independent properties over ALL envs: every column is ceiling* band*
  floor* (the row classification is monotone), band pixels carry one depth
  and one semantic per column, plane pixels the row's plane depth/semantic,
  depth in (0, max_range], semantics from {0, 65534, 65535} or the scene's
  ids, and a rerun from the same state is bit-identical (determinism).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEPTH_RTOL = 1e-5
RGB_ATOL = 1.0 / 255.0 + 1e-9
POSE_ATOL = 1e-6


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_01201_b200 as nb
    from paper_1904_01201_b200 import _native
    _native.load()
    return nb


def _check_batch(nb, oracle_mod, cfg, N, W, H, steps, n_sample, seed):
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene(cfg)
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("semantic", W, H))
    sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, N, sensor_configs=suite,
                            floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
    poses = synth.sample_poses(sc, N, seed=seed)
    sim.reset(poses[:, :2], poses[:, 2])
    acts = synth.random_actions(N, steps, seed=seed + 1)
    osc = oracle_mod.OracleScene(sc.segments, sc.semantic_ids, sc.albedo, sc.wall_height,
                                 sc.floor_color, sc.ceiling_color)
    rng = np.random.default_rng(seed + 2)
    sample = rng.choice(N, size=min(n_sample, N), replace=False)
    states = {int(e): [poses[e, 0], poses[e, 1], oracle_mod.wrap_angle(poses[e, 2]), 0.0, 0]
              for e in sample}
    focal = suite[0].focal
    valid_sem = np.union1d(np.unique(sc.semantic_ids), [0, 65534, 65535]).astype(np.int64)
    for s in range(acts.shape[0]):
        sim.step(torch.as_tensor(acts[s], device="cuda:0"))
        torch.cuda.synchronize()
        obs = sim.observations()
        xy, h, _, _ = (v.cpu().numpy() for v in sim.state())
        dep = obs["depth"]
        sem = obs["semantic"].to(torch.int64) if obs["semantic"].dtype != torch.uint16 else \
            obs["semantic"].view(torch.int16).to(torch.int64) & 0xFFFF
        # --- properties over all envs (device-side reductions)
        assert bool((dep > 0).all()) and bool((dep <= 10.0).all())
        assert bool(torch.isin(sem.unique(), torch.as_tensor(valid_sem, device=sem.device)).all())
        ceil = sem == 65535
        floor = sem == 65534
        band = ~(ceil | floor)
        # ceiling rows form a prefix, floor rows a suffix of every column
        assert bool((ceil[:, 1:, :] <= ceil[:, :-1, :]).all())
        assert bool((floor[:, 1:, :] >= floor[:, :-1, :]).all())
        assert bool((band.int().diff(dim=1).abs().sum(dim=1) <= 2).all())
        # one depth and one semantic per column inside the band
        dmax = torch.where(band, dep, torch.full_like(dep, -1.0)).amax(dim=1)
        dmin = torch.where(band, dep, torch.full_like(dep, 1e9)).amin(dim=1)
        has = band.any(dim=1)
        assert bool((dmax[has] == dmin[has]).all())
        # plane pixels: the row's plane depth is the same for every env/column
        for plane in (ceil, floor):
            row_max = torch.where(plane, dep, torch.full_like(dep, -1.0)).amax(dim=(0, 2))
            row_min = torch.where(plane, dep, torch.full_like(dep, 1e9)).amin(dim=(0, 2))
            rows = plane.any(dim=2).any(dim=0)
            assert bool((row_min[rows] == row_max[rows]).all())
        # --- sampled envs vs the oracle
        rgb_h, dep_h, sem_h = obs["rgb"].cpu().numpy(), dep.cpu().numpy(), \
            obs["semantic"].cpu().numpy()
        for e in sample:
            e = int(e)
            states[e], _, _ = osc.step(states[e], int(acts[s, e]))
            st = states[e]
            assert abs(xy[e, 0] - st[0]) <= POSE_ATOL and abs(xy[e, 1] - st[1]) <= POSE_ATOL
            assert abs(h[e] - st[2]) <= POSE_ATOL
            rgb, d, smn = osc.render((xy[e, 0], xy[e, 1]), h[e], 1.5, W, H, focal=focal)
            assert np.array_equal(sem_h[e], smn), (s, e)
            rel = np.abs(dep_h[e].astype(np.float64) - d) / np.maximum(np.abs(d), 1e-12)
            assert rel.max() <= DEPTH_RTOL
            assert np.abs(rgb_h[e].astype(np.float64) / 255.0 - rgb).max() <= RGB_ATOL
    return sim


def test_c3_fullsize(nb, oracle_mod):
    sim = _check_batch(nb, oracle_mod, "C3", 1024, 256, 256, steps=4, n_sample=12, seed=41)
    # determinism: render again from the same state -> identical frames
    first = {k: v.clone() for k, v in sim.observations().items()}
    sim.render()
    torch.cuda.synchronize()
    again = sim.observations()
    for k in first:
        assert torch.equal(first[k].view(torch.uint8), again[k].view(torch.uint8))


def test_c5_fullsize(nb, oracle_mod):
    """C5 at full per-GPU size: 512 envs x 512x512 on the ~1M-triangle scene,
    a seeded sample of envs against the oracle at every step."""
    _check_batch(nb, oracle_mod, "C5", 512, 512, 512, steps=3, n_sample=10, seed=51)


def test_c5_small_batch_every_env(nb, oracle_mod):
    """C5's scene and resolution with every env compared at every step (8 envs
    x 6 steps: the warp-per-ray cast and the row-banded writer)."""
    _check_batch(nb, oracle_mod, "C5", 8, 512, 512, steps=6, n_sample=8, seed=61)
