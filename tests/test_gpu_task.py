"""Parity of the CUDA navigation / task row (nv_nav_* / nv_task_*, SURVEY §8f
rows 1-2) with the reference, through the C ABI:

* occupancy masks, wall clearances, goal snapping, distance fields and
  geodesic queries bit-exact against fixtures produced by the unmodified
  reference (tests/golden/make_golden_task.py);
* whole PointGoal episodes (per-step distance, reward, done flag, collision,
  displacement and pose, final EpisodeOutcome) bit-exact, all episodes of a
  scene stepped together as one batch;
* larger grids (the C2 apartment) against the live oracle
  (oracle/navsim_nav_oracle.c, pinned to the same fixtures).
"""
import glob
import hashlib
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FILES = sorted(glob.glob(os.path.join(HERE, "golden", "golden_task_*.npz")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_01201_b200 as nb
    from paper_1904_01201_b200 import _native
    _native.load()
    return nb


@pytest.fixture(scope="module", params=FILES, ids=[os.path.basename(f)[12:-4] for f in FILES])
def gold(request):
    return dict(np.load(request.param))


def grid_for(nb, gold, radius):
    from paper_1904_01201_b200 import nav
    return nav.rasterize_navigable(gold["segments"], tuple(gold["bounds"]), 0.05, radius)


def test_grid_exact(nb, gold):
    for key in [k[:-7] for k in gold if k.endswith("_origin")]:
        r = int(key[1:]) / 1000.0
        g = grid_for(nb, gold, r)
        assert np.array_equal(g.origin, gold[f"{key}_origin"])
        assert np.array_equal(g.navigable.astype(np.uint8), gold[f"{key}_navigable"]), key
        assert np.array_equal(g.clearance.ravel()[gold[f"{key}_clearance_idx"]],
                              gold[f"{key}_clearance_val"])
        assert sha(g.clearance) == str(gold[f"{key}_clearance_sha"])


def test_snap_fields_geodesic_exact(nb, gold):
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import nav
    g = grid_for(nb, gold, 0.1)
    cells = g.snap(gold["snap_pts"])
    assert np.array_equal(cells, gold["snap_cells"].astype(np.int32))
    fields, fc = nav.distance_fields(g, gold["field_goal"])
    assert np.array_equal(fc, gold["field_cell"].astype(np.int32))
    host = fields.cpu().numpy()
    for k in range(len(gold["field_goal"])):
        assert np.array_equal(host[k].ravel()[gold["field_idx"][k]], gold["field_val"][k])
        assert sha(host[k]) == str(gold["field_sha"][k])
    # geodesic queries, all fields at once through nv_nav_geodesic
    pts = torch.as_tensor(gold["geo_pts"].reshape(-1, 2), device="cuda:0")
    fid = torch.as_tensor(np.repeat(np.arange(len(gold["field_goal"]), dtype=np.int32),
                                    gold["geo_pts"].shape[1]), device="cuda:0")
    out = torch.empty(pts.shape[0], dtype=torch.float64, device="cuda:0")
    c = g.ctx
    nat.check(c.lib.nv_nav_geodesic(c.handle, nat.ptr(fields), nat.ptr(fid), nat.ptr(pts),
                                     pts.shape[0], nat.ptr(out), nat.stream_handle("cuda:0")))
    got = out.cpu().numpy()
    want = gold["geo_val"].reshape(-1)
    both_nan = np.isnan(got) & np.isnan(want)
    assert np.array_equal(got[~both_nan], want[~both_nan])


# nv_task_step_render with the task riding on the warp / thread cast, or
# step + nv_task_step
@pytest.mark.parametrize("path", ["cast-warp", "cast-thread", "separate"])
def test_episodes_batched_exact(nb, gold, path):
    if "n_episodes" not in gold:
        pytest.skip("no episodes in this fixture")
    from paper_1904_01201_b200 import task
    from paper_1904_01201_b200.sensors import SensorConfig
    n = int(gold["n_episodes"])
    segs = gold["segments"]
    ns = len(segs)
    env = task.BatchEnvironment((segs, np.arange(1, ns + 1, dtype=np.uint16), np.full((ns, 3), 0.5)),
                                n, sensor_configs=(SensorConfig("depth", width=64, height=16),))
    from paper_1904_01201_b200 import _native as nat
    env.fused_task = path != "separate"
    mode = {"cast-warp": nat.NV_CAST_WARP, "cast-thread": nat.NV_CAST_THREAD,
            "separate": nat.NV_CAST_AUTO}[path]
    nat.check(env.sim.ctx.lib.nv_set_cast_mode(env.sim.ctx.handle, mode))
    eps = []
    for k in range(n):
        p = f"ep{k}_"
        sr, goal = gold[p + "start_raw"], gold[p + "goal"]
        gd = float(gold[p + "gdsp"])
        eu = math.hypot(goal[0] - sr[0], goal[1] - sr[1])
        eps.append(task.Episode(f"e{k}", "x", (float(sr[0]), float(sr[1])), float(sr[2]),
                                (float(goal[0]), float(goal[1])), gd, eu, gd / eu))
    env.reset(eps)
    assert np.array_equal(env.d0, np.array([float(gold[f"ep{k}_d0"]) for k in range(n)]))
    xy, h, _, _ = env.sim.state()
    for k in range(n):
        st = gold[f"ep{k}_start"]
        assert xy[k, 0].item() == st[0] and xy[k, 1].item() == st[1] and h[k].item() == st[2]
    T = max(len(gold[f"ep{k}_actions"]) for k in range(n))
    acts = np.zeros((T, n), dtype=np.int8)
    for k in range(n):
        a = gold[f"ep{k}_actions"]
        acts[: len(a), k] = a
    for t in range(T):
        _, done, info = env.step(torch.as_tensor(acts[t], device="cuda:0"))
        torch.cuda.synchronize()
        xy, h, _, _ = env.sim.state()
        d, r = info["d"].cpu().numpy(), info["reward"].cpu().numpy()
        dn, co = done.cpu().numpy(), info["collided"].cpu().numpy()
        mv, stt = info["displacement"].cpu().numpy(), info["status"].cpu().numpy()
        xy, h = xy.cpu().numpy(), h.cpu().numpy()
        for k in range(n):
            rows = gold[f"ep{k}_rows"]
            if t < len(rows):
                row = rows[t]
                assert (d[k], r[k], float(dn[k]), float(co[k]), mv[k]) == tuple(row[:5]), (k, t)
                assert (xy[k, 0], xy[k, 1], h[k]) == tuple(row[5:8]), (k, t)
            else:
                # NV_ENV_DONE: frozen; a finished env earns nothing more and
                # keeps its last distance (no terminal reward counted twice)
                assert stt[k] == 4 and dn[k] == 1
                assert r[k] == 0.0 and d[k] == rows[-1][0], (k, t)
    outs = env.outcomes()
    for k in range(n):
        o = gold[f"ep{k}_outcome"]
        got = outs[k]
        assert got is not None
        assert (float(got.success), got.shortest_path, got.path_taken, got.spl, float(got.steps),
                float(got.collisions), 1.0 if got.terminated_by == "stop" else 2.0) == tuple(o)


def test_single_env_facade_matches_batch(nb):
    """task.Environment (reference API over a one-env batch) on the square scene."""
    from paper_1904_01201_b200 import scene as sm
    from paper_1904_01201_b200 import task
    from paper_1904_01201_b200.sim import Action
    g = dict(np.load(os.path.join(HERE, "golden", "golden_task_square.npz")))
    walls = [sm.WallSegment(a=(s[0], s[1]), b=(s[2], s[3]), semantic_id=k + 1,
                            albedo=(0.5, 0.5, 0.5)) for k, s in enumerate(g["segments"])]
    scene = sm.Scene(id="square-10", walls=walls, floor_color=(0.3, 0.3, 0.3),
                     ceiling_color=(0.9, 0.9, 0.9))
    env = task.Environment(scene)
    sr, goal, gd = g["ep0_start_raw"], g["ep0_goal"], float(g["ep0_gdsp"])
    eu = math.hypot(goal[0] - sr[0], goal[1] - sr[1])
    ep = task.Episode("e0", "square-10", (sr[0], sr[1]), sr[2], (goal[0], goal[1]), gd, eu, gd / eu)
    codes = [Action.MOVE_FORWARD, Action.TURN_LEFT, Action.TURN_RIGHT, Action.STOP]
    out = task.run_episode(env, ep, [codes[int(a)] for a in g["ep0_actions"]])
    o = g["ep0_outcome"]
    assert (float(out.success), out.path_taken, out.spl, float(out.steps)) == (o[0], o[2], o[3], o[4])
    with pytest.raises(task.TaskError):
        env.step(Action.STOP)
    bad = task.Episode("e1", "other", (sr[0], sr[1]), sr[2], (goal[0], goal[1]), gd, eu, gd / eu)
    with pytest.raises(task.TaskError):
        env.reset(bad)


def test_apartment_fields_vs_oracle(nb):
    """C2 apartment (10k segments): device grid + fields bit-exact vs the oracle."""
    from oracle import nav_oracle as no
    from paper_1904_01201_b200 import nav, synth
    sc = synth.config_scene("C2")
    bnds = no.bounds(sc.segments)
    g = nav.rasterize_navigable(sc.segments, bnds)
    og = no.Grid(sc.segments, bnds)
    assert np.array_equal(g.navigable.astype(np.uint8), og.navigable)
    assert np.array_equal(g.clearance, og.clearance)
    rng = np.random.default_rng(3)
    cells = np.argwhere(og.navigable)
    goals = [og.center_of(*cells[int(rng.integers(len(cells)))]) for _ in range(3)]
    fields, fc = nav.distance_fields(g, goals)
    host = fields.cpu().numpy()
    for k, goal in enumerate(goals):
        assert tuple(fc[k]) == og.snap(goal)
        assert np.array_equal(host[k], og.field(tuple(fc[k])))


def test_envs_realloc_drops_task_state(nb, gold):
    """nv_envs_alloc after PointGoal episodes (here: a larger batch) starts
    from un-reset, un-frozen envs: no stale done flag freezes the new envs
    and the task buffers of the old batch are never read (nv_task_step
    refuses until nv_task_reset)."""
    if "n_episodes" not in gold:
        pytest.skip("no episodes in this fixture")
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import task
    from paper_1904_01201_b200.sensors import SensorConfig
    n = int(gold["n_episodes"])
    segs = gold["segments"]
    ns = len(segs)
    env = task.BatchEnvironment((segs, np.arange(1, ns + 1, dtype=np.uint16), np.full((ns, 3), 0.5)),
                                n, sensor_configs=(SensorConfig("depth", width=64, height=16),))
    eps = []
    for k in range(n):
        p = f"ep{k}_"
        sr, goal = gold[p + "start_raw"], gold[p + "goal"]
        gd = float(gold[p + "gdsp"])
        eu = math.hypot(goal[0] - sr[0], goal[1] - sr[1])
        eps.append(task.Episode(f"e{k}", "x", (float(sr[0]), float(sr[1])), float(sr[2]),
                                (float(goal[0]), float(goal[1])), gd, eu, gd / eu))
    env.reset(eps)
    _, done, _ = env.step(torch.full((n,), 3, dtype=torch.int8, device="cuda:0"))  # STOP: all done
    assert bool(done.all())
    c = env.sim.ctx
    m = 4 * n + 3
    nat.check(c.lib.nv_envs_alloc(c.handle, m))
    xy = np.ascontiguousarray(np.repeat(gold["ep0_start"][None, :2], m, axis=0))
    hd = np.full(m, float(gold["ep0_start"][2]))
    st = np.zeros(m, dtype=np.int32)
    nat.check(c.lib.nv_set_poses(c.handle, nat.ptr(xy), nat.ptr(hd), None, nat.ptr(st), None))
    acts = torch.zeros(m, dtype=torch.int8, device="cuda:0")
    status = torch.full((m,), -1, dtype=torch.int32, device="cuda:0")
    nat.check(c.lib.nv_step(c.handle, nat.ptr(acts), None, None, nat.ptr(status),
                            nat.stream_handle("cuda:0")))
    torch.cuda.synchronize()
    assert bool((status == 0).all())
    assert c.lib.nv_task_step(c.handle, nat.ptr(acts), nat.ptr(status), None, None, None, None,
                              None) == nat.NV_ERR_STATE


def test_depth_noise_moments_and_paths(nb):
    """Inverse-depth noise (nv_depth_noise, sensors.py:183-205): the reference's
    moment test on the device stream (eps = max_range/d' - max_range/d has std
    sigma), saturated pixels untouched, clamping, determinism, and the same
    noisy frame from every fill path (fused in the ws writer, a pass
    otherwise)."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C2")
    W = H = 128
    n = 48
    suite = (nb.SensorConfig("depth", W, H),)
    sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
    poses = synth.sample_poses(sc, n, seed=12)
    sim.reset(poses[:, :2], poses[:, 2])
    c = sim.ctx
    sim.render()
    torch.cuda.synchronize()
    clean = sim.observations()["depth"].clone().double()
    outs = []
    for mode in (nat.NV_FILL_AUTO, nat.NV_FILL_GENERIC):
        nat.check(c.lib.nv_set_fill_mode(c.handle, mode))
        nat.check(c.lib.nv_depth_noise(c.handle, 0.4, 1234, 0))
        sim.render()
        torch.cuda.synchronize()
        outs.append(sim.observations()["depth"].clone())
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    noisy = outs[0].double()
    mr = 10.0
    void = clean >= mr
    assert torch.equal(noisy[void], clean[void])
    live = ~void
    assert noisy[live].min().item() >= 0.05 - 1e-7 and noisy[live].max().item() <= mr
    sel = (clean <= 4.0) & (noisy > 0.05) & (noisy < mr)
    eps = (mr / noisy[sel] - mr / clean[sel]).cpu().numpy()
    assert eps.size > 100000
    assert abs(eps.mean()) < 0.01
    assert eps.std() == pytest.approx(0.4, abs=0.01)
    # a new seed changes the frame; the same seed reproduces it
    nat.check(c.lib.nv_depth_noise(c.handle, 0.4, 1234, 0))
    sim.render()
    torch.cuda.synchronize()
    assert torch.equal(sim.observations()["depth"], outs[0])
    nat.check(c.lib.nv_depth_noise(c.handle, 0.4, 99, 0))
    sim.render()
    torch.cuda.synchronize()
    assert not torch.equal(sim.observations()["depth"], outs[0])
    assert c.lib.nv_depth_noise(c.handle, -1.0, 0, 0) == nat.NV_ERR_ARG


def test_apartment_batch_episodes_vs_oracle(nb):
    """256 PointGoal envs on the C2 apartment (10k segments) through
    BatchEnvironment vs the oracle's Environment restatement on a sample of
    envs: per-step distance, reward, done and pose, and the outcomes --
    bit-exact."""
    import math
    from oracle import nav_oracle as no
    from oracle import oracle as orc
    from paper_1904_01201_b200 import synth, task
    from paper_1904_01201_b200.sensors import SensorConfig
    sc = synth.config_scene("C2")
    segs = sc.segments
    bnds = no.bounds(segs)
    og = no.Grid(segs, bnds)
    N = 256
    env = task.BatchEnvironment((segs, sc.semantic_ids, sc.albedo), N,
                                sensor_configs=(SensorConfig("depth", 64, 16),))
    rng = np.random.default_rng(12)
    cells = np.argwhere(og.navigable)
    eps, starts, goals = [], [], []
    while len(eps) < N:
        s = og.center_of(*cells[int(rng.integers(len(cells)))])
        g = og.center_of(*cells[int(rng.integers(len(cells)))])
        eu = math.hypot(*(g - s))
        if not (1.5 <= eu <= 6.0):
            continue
        eps.append(task.Episode(f"e{len(eps)}", "x", (float(s[0]), float(s[1])),
                                float(rng.uniform(-math.pi, math.pi)), (float(g[0]), float(g[1])),
                                max(1.0, eu), eu, max(1.0, eu) / eu))
    env.reset(eps)
    sample = rng.choice(N, size=6, replace=False)
    scene = orc.OracleScene(segs, sc.semantic_ids, sc.albedo)
    oenv = {int(e): no.TaskEnv(scene, og) for e in sample}
    for e, oe in oenv.items():
        ep = eps[e]
        d0 = oe.reset(ep.start_position, ep.start_heading, ep.goal_position, ep.gdsp)
        assert d0 == env.d0[e]
    T = 60
    acts = rng.choice(3, size=(T, N), p=[0.6, 0.2, 0.2]).astype(np.int8)
    acts[T - 1] = 3  # everyone stops
    done_o = {e: False for e in oenv}
    for t in range(T):
        _, done, info = env.step(torch.as_tensor(acts[t], device="cuda:0"))
        torch.cuda.synchronize()
        d, r = info["d"].cpu().numpy(), info["reward"].cpu().numpy()
        dn = done.cpu().numpy()
        xy, h, _, _ = (v.cpu().numpy() for v in env.sim.state())
        for e, oe in oenv.items():
            if done_o[e]:
                continue
            dd, rr, ddone, _, _, out = oe.step(int(acts[t, e]))
            assert (d[e], r[e], bool(dn[e])) == (dd, rr, ddone), (t, e)
            assert (xy[e, 0], xy[e, 1], h[e]) == tuple(oe.state[:3])
            done_o[e] = ddone
    outs = env.outcomes()
    assert all(o is not None for o in outs)


def test_rebuilt_grid_invalidates_old_grid_objects(nb):
    """A context holds one navigation grid: after a rebuild with other bounds,
    the old OccupancyGrid refuses host copies / snaps (its sizes no longer
    match the device buffers) and nv_nav_copy refuses mismatched buffers."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import nav, synth
    sc = synth.single_room(20)
    g1 = nav.rasterize_navigable(sc.segments, (0.0, 0.0, 10.0, 10.0))
    assert g1.navigable.shape == (g1.height, g1.width)
    g2 = nav.build_grid(g1.ctx, (0.0, 0.0, 5.0, 10.0))
    assert (g2.width, g2.height) != (g1.width, g1.height)
    with pytest.raises(nav.NavError):
        _ = g1.clearance if not g1._host else nav.distance_fields(g1, [(2.0, 2.0)])
    with pytest.raises(nav.NavError):
        g1.snap([(2.0, 2.0)])
    assert g2.navigable.shape == (g2.height, g2.width)
    m = np.empty((g1.height, g1.width), np.uint8)
    rc = g1.ctx.lib.nv_nav_copy(g1.ctx.handle, g1.width, g1.height, nat.ptr(m), None)
    assert rc == nat.NV_ERR_STATE


def test_task_steps_overlap_agrees_at_scale(nb):
    """The task-layer step with the cast -> writer release and the chained
    agent step (thread-per-ray batch: 512 envs x 128 columns) gives the same
    rewards, distances, done flags, poses, frames and EpisodeOutcome records
    as the serialised launches (nv_set_overlap 0), bit for bit."""
    import math
    from oracle import nav_oracle as no
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth, task
    from paper_1904_01201_b200.sensors import SensorConfig
    sc = synth.config_scene("C2")
    segs = sc.segments
    og = no.Grid(segs, no.bounds(segs))
    N, T = 512, 24
    rng = np.random.default_rng(33)
    cells = np.argwhere(og.navigable)
    eps = []
    while len(eps) < N:
        s = og.center_of(*cells[int(rng.integers(len(cells)))])
        g = og.center_of(*cells[int(rng.integers(len(cells)))])
        eu = math.hypot(*(g - s))
        if not (1.5 <= eu <= 6.0):
            continue
        eps.append(task.Episode(f"e{len(eps)}", "x", (float(s[0]), float(s[1])),
                                float(rng.uniform(-math.pi, math.pi)), (float(g[0]), float(g[1])),
                                max(1.0, eu), eu, max(1.0, eu) / eu))
    acts = rng.choice(3, size=(T, N), p=[0.6, 0.2, 0.2]).astype(np.int8)
    acts[T - 1] = 3
    envs = []
    for overlap in (0, 1):
        env = task.BatchEnvironment((segs, sc.semantic_ids, sc.albedo), N,
                                    sensor_configs=(SensorConfig("rgb", 128, 32),
                                                    SensorConfig("depth", 128, 32)))
        nat.check(env.sim.ctx.lib.nv_set_overlap(env.sim.ctx.handle, overlap))
        env.reset(eps)
        envs.append(env)
    for t in range(T):
        outs = []
        for env in envs:
            obs, done, info = env.step(torch.as_tensor(acts[t], device="cuda:0"))
            torch.cuda.synchronize()
            outs.append((done.clone(), info["d"].clone(), info["reward"].clone(),
                         [v.clone() for v in env.sim.state()],
                         {k: v.clone() for k, v in env.sim.observations().items()}))
        (d0, dd0, r0, s0, o0), (d1, dd1, r1, s1, o1) = outs
        assert torch.equal(d0, d1) and torch.equal(dd0, dd1) and torch.equal(r0, r1), t
        for a, b in zip(s0, s1):
            assert torch.equal(a, b), t
        for k in o0:
            assert torch.equal(o0[k], o1[k]), (t, k)
    assert envs[0].outcomes() == envs[1].outcomes()
    assert envs[1].sim.ctx.faults() == 0  # no handshake wait gave up
