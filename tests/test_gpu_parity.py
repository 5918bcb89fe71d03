"""Parity of the CUDA path (through the C ABI) with the reference.

* golden fixtures (produced by the unmodified reference, tests/golden/) for
  the operator-level entry points: raycast (bit-exact), fill_frame (semantic
  and coverage exact, depth 1e-5 rel, RGB 1/255), disc casts / clearance
  (bit-exact), kinematics episodes (poses 1e-6);
* the live oracle (C restatement pinned to the same fixtures) for the batched
  device path at sizes the oracle finishes in seconds.

Tolerances are the north-star's: semantic ids and pixel coverage bit-exact,
depth within 1e-5 relative, RGB within 1/255 per channel, poses within 1e-6.
"""
import math

import numpy as np
import pytest

from conftest import golden_names, load_golden

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


def geom_of(nb, g):
    return nb.RenderGeometry(g["segments"], g["semantic_ids"], g["albedo"], float(g["wall_height"]),
                             g["floor_color"], g["ceiling_color"])


def check_frame(rgb_u8, dep_f32, sem, ref_rgb, ref_dep, ref_sem, ctx=""):
    """rgb_u8 (H,W,3) u8, dep_f32 (H,W) f32, sem (H,W) u16 vs reference f64/u16."""
    assert np.array_equal(sem, ref_sem), f"{ctx}: semantic mismatch at " \
        f"{np.argwhere(sem != ref_sem)[:5].tolist()}"
    d = dep_f32.astype(np.float64)
    rel = np.abs(d - ref_dep) / np.maximum(np.abs(ref_dep), 1e-12)
    assert rel.max() <= DEPTH_RTOL, f"{ctx}: depth rel err {rel.max()}"
    err = np.abs(rgb_u8.astype(np.float64) / 255.0 - ref_rgb)
    assert err.max() <= RGB_ATOL, f"{ctx}: rgb err {err.max() * 255:.3f}/255"


@pytest.mark.parametrize("name", golden_names())
def test_raycast_bit_exact(nb, name):
    g = load_golden(name)
    geom = geom_of(nb, g)
    for k, (x, y, _) in enumerate(g["poses"]):
        t, i = geom.index.raycast((x, y), g["cast_dirs"][k])
        assert np.array_equal(i, g["cast_i_grid"][k])
        assert np.array_equal(t, g["cast_t_grid"][k])
        t, i = geom.index.raycast_brute((x, y), g["cast_dirs"][k])
        assert np.array_equal(i, g["cast_i_brute"][k])
        assert np.array_equal(t, g["cast_t_brute"][k])


@pytest.mark.parametrize("name", golden_names())
def test_grid_matches_reference(nb, name):
    g = load_golden(name)
    geom = geom_of(nb, g)
    idx = geom.index
    assert (idx.x0, idx.y0, idx.nx, idx.ny) == (g["grid_x0"], g["grid_y0"], g["grid_nx"],
                                                 g["grid_ny"])
    assert idx.n_items == len(g["grid_items"])


@pytest.mark.parametrize("name", golden_names())
def test_render_facade_vs_golden(nb, name):
    """sensors.render on the GPU vs the reference's frames (fixtures)."""
    g = load_golden(name)
    geom = geom_of(nb, g)
    keys = sorted(k[:-len("_focal")] for k in g if k.startswith("frame_") and k.endswith("_focal"))
    for key in keys:
        w, h = (int(v) for v in key[len("frame_"):].split("x"))
        suite = (nb.SensorConfig("rgb", w, h), nb.SensorConfig("depth", w, h),
                 nb.SensorConfig("semantic", w, h))
        for k, (x, y, hd) in enumerate(g["poses"]):
            dev = nb.sensors.render_device(geom, (x, y), hd, float(g["sensor_height"]), suite)
            check_frame(dev["rgb"].cpu().numpy(), dev["depth"].cpu().numpy(),
                        dev["semantic"].cpu().numpy(), g[key + "_rgb_f32"][k].astype(np.float64),
                        g[key + "_depth_f32"][k].astype(np.float64), g[key + "_sem"][k],
                        f"{name} {key} pose {k}")
            # brute-force index gives the identical frame (tests/test_sensors.py:186-199)
            devb = nb.sensors.render_device(geom, (x, y), hd, float(g["sensor_height"]), suite,
                                            brute_force=True)
            assert torch.equal(devb["semantic"].view(torch.int16), dev["semantic"].view(torch.int16))
            assert torch.equal(devb["depth"], dev["depth"])
            assert torch.equal(devb["rgb"], dev["rgb"])


@pytest.mark.parametrize("name", golden_names())
def test_disc_cast_and_clearance_bit_exact(nb, name):
    g = load_golden(name)
    geom = geom_of(nb, g)
    q = g["disc_queries"]
    t, seg, tan = geom.index.cast_disc_batch(q[:, 0], q[:, 1], q[:, 2], q[:, 3], q[:, 4])
    res = g["disc_results"]
    assert np.array_equal(seg.astype(np.float64), res[:, 1])
    assert np.array_equal(t, res[:, 0])
    assert np.array_equal(tan, res[:, 2:4])
    clr = geom.index.clearance_batch(q[:, 0], q[:, 1])
    assert np.array_equal(clr, g["clearance"])


@pytest.mark.parametrize("name", [n for n in golden_names() if n != "rand120"])
def test_batch_kinematics_vs_golden(nb, name):
    """Batched device Simulator.step over the reference's recorded episodes."""
    g = load_golden(name)
    starts = g["kin_starts"]
    if len(starts) == 0:
        pytest.skip("no episodes")
    E = len(starts)
    sim = nb.BatchSimulator(g["segments"], g["semantic_ids"], g["albedo"], E, sensor_configs=(),
                            wall_height=float(g["wall_height"]))
    sim.reset(starts[:, :2], starts[:, 2])
    acts = torch.as_tensor(g["kin_actions"].T.copy(), device="cuda:0")  # (steps, E)
    exact = 0
    for s in range(acts.shape[0]):
        sim.step(acts[s].contiguous(), render=False)
        xy, h, p, k = (v.cpu().numpy() for v in sim.state())
        ref = g["kin_states"][:, s]
        assert np.all(np.abs(xy[:, 0] - ref[:, 0]) <= POSE_ATOL), (name, s)
        assert np.all(np.abs(xy[:, 1] - ref[:, 1]) <= POSE_ATOL), (name, s)
        assert np.all(np.abs(h - ref[:, 2]) <= POSE_ATOL), (name, s)
        assert np.all(np.abs(p - ref[:, 3]) <= POSE_ATOL), (name, s)
        assert np.array_equal(k, ref[:, 4].astype(np.int64)), (name, s)
        coll = sim.collided.cpu().numpy().astype(bool)
        assert np.array_equal(coll, g["kin_collided"][:, s]), (name, s)
        exact += int(np.all(xy[:, 0] == ref[:, 0]) and np.all(xy[:, 1] == ref[:, 1]))
    print(f"{name}: {exact}/{acts.shape[0]} steps bit-identical poses")


def _oracle_scene(oracle, sc):
    return oracle.OracleScene(sc.segments, sc.semantic_ids, sc.albedo, sc.wall_height,
                              sc.floor_color, sc.ceiling_color)


@pytest.mark.parametrize("cfg,W,H,n_envs,steps", [
    ("C1", 64, 48, 16, 40),        # TMA path W=64
    ("C2", 128, 128, 16, 25),      # TMA path W=128 (depth-only config's scene)
    ("C3", 256, 256, 8, 6),        # TMA path W=256, ~100k segments
    ("C1", 40, 33, 8, 20),         # generic path, odd H
])
# cast: auto (warp per ray at these small batches), thread per ray, thread per
# ray overlapped with the agent step (programmatic dependent launch, per-env
# ready flags), warp per ray overlapped
@pytest.mark.parametrize("cast_mode", ["auto", "thread", "thread-overlap", "warp-overlap"])
def test_batch_step_render_vs_oracle(nb, oracle_mod, cfg, W, H, n_envs, steps, cast_mode):
    """Batched step+render (device cos/sin, device DDA, TMA fill) vs the oracle
    run on the same actions: poses 1e-6, frames at the stated tolerances."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene(cfg)
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("semantic", W, H), nb.SensorConfig("gps_compass"))
    sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n_envs, sensor_configs=suite,
                            floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
    nat.check(sim.ctx.lib.nv_set_cast_mode(
        sim.ctx.handle, {"auto": nat.NV_CAST_AUTO, "thread": nat.NV_CAST_THREAD,
                         "thread-overlap": nat.NV_CAST_THREAD,
                         "warp-overlap": nat.NV_CAST_WARP}[cast_mode]))
    nat.check(sim.ctx.lib.nv_set_overlap(sim.ctx.handle, int(cast_mode.endswith("overlap"))))
    poses = synth.sample_poses(sc, n_envs, seed=17)
    sim.reset(poses[:, :2], poses[:, 2])
    acts = synth.random_actions(n_envs, steps, seed=5)
    osc = _oracle_scene(oracle_mod, sc)
    states = [[p[0], p[1], oracle_mod.wrap_angle(p[2]), 0.0, 0] for p in poses]
    focal = suite[0].focal
    for s in range(steps):
        sim.step(torch.as_tensor(acts[s], device="cuda:0"))
        obs = {k: v.cpu().numpy() for k, v in sim.observations().items()}
        xy, h, _, _ = (v.cpu().numpy() for v in sim.state())
        for e in range(n_envs):
            states[e], _, _ = osc.step(states[e], int(acts[s, e]))
            st = states[e]
            assert abs(xy[e, 0] - st[0]) <= POSE_ATOL and abs(xy[e, 1] - st[1]) <= POSE_ATOL
            assert abs(h[e] - st[2]) <= POSE_ATOL
            if s % max(1, steps // 4) == 0 or s == steps - 1:
                # render the oracle at the DEVICE pose so frame parity is not
                # conflated with (tolerated) sub-ulp pose differences
                rgb, dep, sem = osc.render((xy[e, 0], xy[e, 1]), h[e], 1.5, W, H, focal=focal)
                check_frame(obs["rgb"][e], obs["depth"][e], obs["semantic"][e], rgb, dep, sem,
                            f"{cfg} step {s} env {e}")
                g, c = oracle_mod.gps_compass(st[0], st[1], st[2], poses[e, 0], poses[e, 1],
                                              oracle_mod.wrap_angle(poses[e, 2]))
                assert np.all(np.abs(obs["gps"][e] - g) <= POSE_ATOL)
                assert abs(obs["compass"][e] - c) <= POSE_ATOL


@pytest.mark.parametrize("W,H", [(256, 64), (128, 40), (512, 32)])
def test_fill_paths_agree(nb, W, H):
    """Identical frames from every frame writer: the warp-specialised TMA
    writer (auto), the per-pixel kernel (forced, and chosen for misaligned
    outputs)."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C2")
    n = 6
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("semantic", W, H))
    sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
    poses = synth.sample_poses(sc, n, seed=3)
    sim.reset(poses[:, :2], poses[:, 2])
    c, st = sim.ctx, nat.stream_handle("cuda:0")
    outs = []
    for mode in (nat.NV_FILL_AUTO, nat.NV_FILL_GENERIC):
        nat.check(c.lib.nv_set_fill_mode(c.handle, mode))
        sim.render()
        torch.cuda.synchronize()
        outs.append({k: v.clone() for k, v in sim.observations().items()})
    raw_rgb = torch.empty(n * H * W * 3 + 1, dtype=torch.uint8, device="cuda:0")
    raw_d = torch.empty(n * H * W + 1, dtype=torch.float32, device="cuda:0")
    raw_s = torch.empty(n * H * W + 1, dtype=torch.int16, device="cuda:0")
    rgb, dep, sem = raw_rgb[1:], raw_d[1:], raw_s[1:]
    nat.check(c.lib.nv_set_fill_mode(c.handle, nat.NV_FILL_AUTO))
    nat.check(c.lib.nv_render(c.handle, 0, nat.ptr(rgb), nat.ptr(dep), nat.ptr(sem), None, None, st))
    torch.cuda.synchronize()
    outs.append({"rgb": rgb.view(n, H, W, 3), "depth": dep.view(n, H, W),
                 "semantic": sem.view(n, H, W).view(torch.uint16)})
    for o in outs[1:]:
        assert torch.equal(o["rgb"], outs[0]["rgb"])
        assert torch.equal(o["depth"], outs[0]["depth"])
        assert torch.equal(o["semantic"].view(torch.int16), outs[0]["semantic"].view(torch.int16))


def test_full_size_properties(nb):
    """C3 at full size (1024 envs, 256^2 RGB-D-S): size-independent properties
    the reference asserts (tests/test_sensors.py:82-89, test_sim.py:146-189):
    depth == max_range <=> semantic == 0, every pixel written, non-penetration
    after stepping, bit-identical reruns."""
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C3")
    n = 1024
    suite = (nb.SensorConfig("rgb"), nb.SensorConfig("depth"), nb.SensorConfig("semantic"))
    poses = synth.sample_poses(sc, n, seed=1)
    acts = torch.as_tensor(synth.random_actions(n, 30, seed=2), device="cuda:0")
    outs = []
    for _ in range(2):
        sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
        sim.reset(poses[:, :2], poses[:, 2])
        for s in range(acts.shape[0]):
            sim.step(acts[s])
        torch.cuda.synchronize()
        o = sim.observations()
        xy, h, _, _ = sim.state()
        outs.append((xy.clone(), h.clone(), o["depth"].clone(), o["semantic"].view(torch.int16).clone(),
                     o["rgb"].clone()))
        dep, sem = o["depth"], o["semantic"].view(torch.int16)
        assert torch.equal(dep == 10.0, sem == 0)
        assert bool(torch.isfinite(dep).all()) and bool((dep > 0).all())
        idx = nb.SegmentIndex(sc.segments)
        clr = idx.clearance_batch(xy[:, 0].cpu().numpy(), xy[:, 1].cpu().numpy())
        assert clr.min() >= 0.1 - 1e-6
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


def test_device_sincos_matches_host(nb):
    """The device agent path's cos/sin are the correctly rounded values the
    host build of the same code returns (exact_math.cuh)."""
    from paper_1904_01201_b200 import _native as nat
    import ctypes
    lib = nat.load()
    rng = np.random.default_rng(0)
    hs = rng.uniform(-math.pi, math.pi, 64)
    sc = np.array([[0.0, 0.0, 100.0, 0.0]])
    n = len(hs)
    sim = nb.BatchSimulator(sc, [1], [[0.5, 0.5, 0.5]], n, sensor_configs=())
    sim.reset(np.stack([np.zeros(n), np.full(n, 50.0)], 1), hs)
    # one forward step moves by step*(cos h, sin h) exactly (free space)
    sim.step(torch.zeros(n, dtype=torch.int8, device="cuda:0"), render=False)
    xy = sim.state()[0].cpu().numpy()
    for e, h in enumerate(hs):
        s, c = ctypes.c_double(), ctypes.c_double()
        lib.nv_host_sincos(nb.wrap_angle(h), ctypes.byref(s), ctypes.byref(c))
        assert xy[e, 0] == 0.0 + 0.25 * c.value
        assert xy[e, 1] == 50.0 + 0.25 * s.value


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_raycast_stress_vs_oracle(nb, oracle_mod, cfg):
    """Random and adversarial rays (aimed exactly at segment endpoints, along
    segments, axis-aligned) through the device DDA (f32 prefilter + exact
    FP64 test) vs the oracle's raycast_grid: bit-identical (t, idx)."""
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene(cfg)
    osc = _oracle_scene(oracle_mod, sc)
    idx = nb.SegmentIndex(sc.segments)
    rng = np.random.default_rng(11)
    poses = synth.sample_poses(sc, 24, seed=99)
    segs = sc.segments
    for (x, y, h) in poses:
        th = rng.uniform(-math.pi, math.pi, 1024)
        dirs = [np.stack([np.cos(th), np.sin(th)], 1)]
        near = segs[np.argsort(np.hypot(segs[:, 0] - x, segs[:, 1] - y))[:256]]
        dirs.append(near[:, 0:2] - [x, y])                  # exactly at endpoints a
        dirs.append(near[:, 2:4] - [x, y])                  # exactly at endpoints b
        dirs.append(near[:, 2:4] - near[:, 0:2])            # parallel to segments
        dirs.append(np.array([[1, 0], [0, 1], [-1, 0], [0, -1], [1, 1], [-1, 1]], float))
        d = np.concatenate(dirs)
        for t_max in (1e9, 10.0):
            tg, ig = idx.raycast((x, y), d, t_max=t_max)
            to, io = osc.raycast((x, y), d, t_max=t_max)
            assert np.array_equal(ig, io)
            assert np.array_equal(tg, to)


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_raycast_prefilter_edges_vs_oracle(nb, oracle_mod, cfg):
    """Cases aimed at the f32 prefilters' error margin and the DDA's integer
    path: origins exactly on cell lines and outside the grid, rays aimed one
    ulp either side of segment endpoints and along cell lines, and origins
    far (>= 2^30 cells) from the grid -- bit-identical (t, idx) to the
    oracle's raycast_grid."""
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene(cfg)
    osc = _oracle_scene(oracle_mod, sc)
    idx = nb.SegmentIndex(sc.segments)
    segs = sc.segments
    rng = np.random.default_rng(5)
    lo = segs[:, :2].min(0).tolist()
    hi = segs[:, :2].max(0).tolist()
    poses = synth.sample_poses(sc, 12, seed=123)
    origins = []
    for (x, y, _) in poses:
        origins += [(x, y), (math.floor(x), y), (x, math.floor(y)), (math.floor(x), math.floor(y))]
    origins += [(lo[0] - 3.25, 0.5 * (lo[1] + hi[1])), (0.5 * (lo[0] + hi[0]), hi[1] + 7.0)]
    for (x, y) in origins:
        near = segs[np.argsort(np.hypot(segs[:, 0] - x, segs[:, 1] - y))[:128]]
        d = []
        for end in (near[:, 0:2], near[:, 2:4]):
            v = end - [x, y]
            d += [v, np.nextafter(v, np.inf), np.nextafter(v, -np.inf),
                  np.stack([np.nextafter(v[:, 0], np.inf), np.nextafter(v[:, 1], -np.inf)], 1)]
        th = rng.uniform(-math.pi, math.pi, 256)
        d.append(np.stack([np.cos(th), np.sin(th)], 1))
        d.append(np.array([[1, 0], [0, 1], [-1, 0], [0, -1]], float))
        d = np.concatenate(d)
        d = d[np.hypot(d[:, 0], d[:, 1]) > 0]
        for t_max in (1e9, 10.0):
            tg, ig = idx.raycast((x, y), d, t_max=t_max)
            to, io = osc.raycast((x, y), d, t_max=t_max)
            assert np.array_equal(ig, io), (x, y, t_max)
            assert np.array_equal(tg, to), (x, y, t_max)
    # far from the grid (>= 2^30 cells): nothing is reachable
    for (x, y) in ((2.0 ** 31, 0.5), (-3e12, 4.0), (10.0, 5e11)):
        d = np.array([[1.0, 0.0], [-1.0, 0.0], [0.3, -0.9], [-0.7, 0.2]])
        tg, ig = idx.raycast((x, y), d, t_max=10.0)
        assert np.all(ig == -1) and np.all(np.isinf(tg))
        to, io = osc.raycast((x, y), d, t_max=10.0)
        assert np.array_equal(ig, io) and np.array_equal(tg, to)


def _graph_from_golden(nb, g):
    walls = [nb.WallSegment(a=(s[0], s[1]), b=(s[2], s[3]), semantic_id=int(i),
                            albedo=tuple(float(c) for c in a))
             for s, i, a in zip(g["segments"], g["semantic_ids"], g["albedo"])]
    sc = nb.Scene(id="golden", walls=walls, floor_color=tuple(g["floor_color"]),
                  ceiling_color=tuple(g["ceiling_color"]), wall_height=float(g["wall_height"]))
    return nb.build_scene_graph(sc)


def test_simulator_facade_matches_reference(nb):
    """The drop-in Simulator (sim.py:133-219 API) replays the reference's
    recorded episode: poses within 1e-6, identical collision flags, reference
    errors raised (tests/test_sim.py:354-409 behaviours)."""
    g = load_golden("square")
    graph = _graph_from_golden(nb, g)
    sim = nb.Simulator(graph, sensor_configs=(nb.SensorConfig("rgb", 64, 48),
                                               nb.SensorConfig("depth", 64, 48),
                                               nb.SensorConfig("gps_compass")))
    with pytest.raises(nb.SimError, match="reset"):
        sim.step(nb.Action.MOVE_FORWARD)
    with pytest.raises(nb.SimError, match="radius"):
        sim.set_agent_state((0.05, 5.0), 0.0)
    x, y, h = g["kin_starts"][0]
    sim.set_agent_state((x, y), h)
    acts = (nb.Action.MOVE_FORWARD, nb.Action.TURN_LEFT, nb.Action.TURN_RIGHT, nb.Action.STOP)
    for s, a in enumerate(g["kin_actions"][0][:120]):
        res, obs = sim.step(acts[int(a)])
        ref = g["kin_states"][0][s]
        assert abs(sim.state.position[0] - ref[0]) <= POSE_ATOL
        assert abs(sim.state.position[1] - ref[1]) <= POSE_ATOL
        assert abs(sim.state.heading - ref[2]) <= POSE_ATOL
        assert res.collided == bool(g["kin_collided"][0][s])
        assert obs.rgb.shape == (48, 64, 3) and obs.rgb.dtype == np.float64
        assert obs.depth.shape == (48, 64) and obs.gps.shape == (2,)
    with pytest.raises(nb.SimError, match="wall height"):
        nb.Simulator(graph, nb.AgentConfig(sensor_height=3.0))


def test_blind_and_gps_only(nb):
    g = load_golden("square")
    graph = _graph_from_golden(nb, g)
    sim = nb.Simulator(graph, sensor_configs=())
    sim.set_agent_state((5.0, 5.0), 0.0)
    _, obs = sim.step(nb.Action.MOVE_FORWARD)
    assert obs.rgb is None and obs.depth is None and obs.gps is None
    sim = nb.Simulator(graph, sensor_configs=(nb.SensorConfig("gps_compass"),))
    sim.set_agent_state((5.0, 5.0), 1.1)
    _, obs = sim.step(nb.Action.MOVE_FORWARD)
    assert np.allclose(obs.gps, [0.25, 0.0], atol=1e-12)   # tests/test_sim.py:412-418
    assert obs.compass == pytest.approx(0.0, abs=1e-12)


@pytest.mark.parametrize("cfg,W,H,n", [("C1", 256, 64, 32), ("C2", 128, 64, 32), ("C3", 256, 32, 64),
                                       ("C1", 40, 33, 16)])
def test_cast_modes_agree(nb, cfg, W, H, n):
    """The per-column DDA by one thread and by one warp per ray give identical
    frames, including the 1000-piece room whose shared endpoints exercise the
    (t, idx) tie rule."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene(cfg)
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("semantic", W, H), nb.SensorConfig("gps_compass"))
    sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite,
                            floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
    poses = synth.sample_poses(sc, n, seed=21)
    sim.reset(poses[:, :2], poses[:, 2])
    acts = torch.as_tensor(synth.random_actions(n, 12, seed=8), device="cuda:0")
    c = sim.ctx
    for s in range(acts.shape[0]):
        sim.step(acts[s], render=False)
        outs = []
        for mode in (nat.NV_CAST_AUTO, nat.NV_CAST_THREAD, nat.NV_CAST_WARP):
            nat.check(c.lib.nv_set_cast_mode(c.handle, mode))
            sim.render()
            torch.cuda.synchronize()
            outs.append({k: v.clone() for k, v in sim.observations().items()})
        for o in outs[1:]:
            assert torch.equal(outs[0]["semantic"].view(torch.int16), o["semantic"].view(torch.int16))
            assert torch.equal(outs[0]["depth"], o["depth"])
            assert torch.equal(outs[0]["rgb"], o["rgb"])
            assert torch.equal(outs[0]["gps"], o["gps"])


@pytest.mark.parametrize("cfg,W,H,n", [("C1", 256, 64, 24), ("C2", 128, 64, 32), ("C1", 40, 33, 16)])
@pytest.mark.parametrize("cast", ["thread", "warp"])
def test_overlap_agrees(nb, cfg, W, H, n, cast):
    """The agent step -> cast overlap (programmatic dependent launch with
    per-env ready flags) gives the same poses, step results and frames as the
    serialised launches over a 10-step random-action episode."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene(cfg)
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("semantic", W, H), nb.SensorConfig("gps_compass"))
    sims = []
    for overlap in (0, 1):
        sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite,
                                floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
        nat.check(sim.ctx.lib.nv_set_cast_mode(
            sim.ctx.handle, nat.NV_CAST_THREAD if cast == "thread" else nat.NV_CAST_WARP))
        nat.check(sim.ctx.lib.nv_set_overlap(sim.ctx.handle, overlap))
        poses = synth.sample_poses(sc, n, seed=5)
        sim.reset(poses[:, :2], poses[:, 2])
        sims.append(sim)
    acts = torch.as_tensor(synth.random_actions(n, 10, seed=9), device="cuda:0")
    for s in range(acts.shape[0]):
        outs = []
        for sim in sims:
            sim.step(acts[s])
            torch.cuda.synchronize()
            o = {k: v.clone() for k, v in sim.observations().items()}
            o["state"] = [t.clone() for t in sim.state()]
            o["step"] = (sim.collided.clone(), sim.displacement.clone(), sim.status.clone())
            outs.append(o)
        for k in ("rgb", "depth", "gps", "compass"):
            assert torch.equal(outs[0][k], outs[1][k]), (s, k)
        assert torch.equal(outs[0]["semantic"].view(torch.int16), outs[1]["semantic"].view(torch.int16))
        for a, b in zip(outs[0]["state"] + list(outs[0]["step"]),
                        outs[1]["state"] + list(outs[1]["step"])):
            assert torch.equal(a, b)


@pytest.mark.parametrize("cfg,W,H,n,steps,mode", [
    ("C3", 256, 256, 512, 24, 0), ("C4", 256, 128, 1024, 16, 0),
    # small batches (writer grids smaller than the GPU: the agent step waits
    # for the previous writer), with the thread-per-ray cast forced (per-env
    # release, pose records, banded writer) and in auto mode (warp casts)
    ("C1", 256, 256, 1, 120, 1), ("C2", 128, 128, 3, 60, 1),
    ("C1", 256, 256, 1, 120, 0), ("C2", 128, 128, 16, 60, 0)])
def test_chained_steps_agree_at_scale(nb, cfg, W, H, n, steps, mode):
    """At batch sizes where the launches really overlap (thread-per-ray cast,
    per-env release into the writer, the next agent step on the previous
    writer's tail, alternating record halves), a multi-step episode gives
    bit-identical frames, poses and step results to the serialised launches
    (nv_set_overlap 0)."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene(cfg)
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("semantic", W, H), nb.SensorConfig("gps_compass"))
    sims = []
    for overlap in (0, 1):
        sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite,
                                floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
        nat.check(sim.ctx.lib.nv_set_overlap(sim.ctx.handle, overlap))
        nat.check(sim.ctx.lib.nv_set_cast_mode(sim.ctx.handle, mode))
        poses = synth.sample_poses(sc, n, seed=21)
        sim.reset(poses[:, :2], poses[:, 2])
        sims.append(sim)
    acts = torch.as_tensor(synth.random_actions(n, steps, seed=22), device="cuda:0")
    # the overlapped simulator runs its steps back to back (no host sync and
    # no other kernel in between, so each agent step chains onto the
    # previous writer); the serial one synchronises after every step
    s0, s1 = sims
    for s in range(steps):
        s1.step(acts[s])
    for s in range(steps):
        s0.step(acts[s])
        torch.cuda.synchronize()
    torch.cuda.synchronize()
    assert s1.ctx.faults() == 0  # no handshake wait gave up
    o0, o1 = s0.observations(), s1.observations()
    for k in ("rgb", "depth", "gps", "compass"):
        assert torch.equal(o0[k], o1[k]), k
    assert torch.equal(o0["semantic"].view(torch.int16), o1["semantic"].view(torch.int16))
    for a, b in zip(s0.state(), s1.state()):
        assert torch.equal(a, b)
    for a, b in zip((s0.collided, s0.displacement, s0.status), (s1.collided, s1.displacement, s1.status)):
        assert torch.equal(a, b)


@pytest.mark.parametrize("cfg,W,H,n,mode", [("C2", 128, 128, 3, 1), ("C1", 256, 256, 1, 1),
                                            ("C2", 128, 128, 16, 0)])
def test_small_batch_chain_repeated(nb, cfg, W, H, n, mode):
    """The chained step at small batches (writer grids smaller than the GPU),
    repeated: eight independent 40-step back-to-back runs must each equal the
    serialised launches (scripts/chain_stress.py found 1 in 15 runs reading a
    stale pose record before the agent step waited for small writer grids)."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene(cfg)
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("gps_compass"))
    steps = 40
    for r in range(8):
        sims = []
        for overlap in (0, 1):
            sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
            nat.check(sim.ctx.lib.nv_set_overlap(sim.ctx.handle, overlap))
            nat.check(sim.ctx.lib.nv_set_cast_mode(sim.ctx.handle, mode))
            poses = synth.sample_poses(sc, n, seed=300 + r)
            sim.reset(poses[:, :2], poses[:, 2])
            sims.append(sim)
        acts = torch.as_tensor(synth.random_actions(n, steps, seed=400 + r), device="cuda:0")
        s0, s1 = sims
        for s in range(steps):
            s1.step(acts[s])
        for s in range(steps):
            s0.step(acts[s])
            torch.cuda.synchronize()
        torch.cuda.synchronize()
        assert s1.ctx.faults() == 0, r
        o0, o1 = s0.observations(), s1.observations()
        for k in ("rgb", "depth", "gps", "compass"):
            assert torch.equal(o0[k], o1[k]), (r, k)
        for a, b in zip(s0.state(), s1.state()):
            assert torch.equal(a, b), r


def test_steps_without_frames_back_to_back(nb):
    """nv_step_render with no frame channels (no writer after the casts),
    issued back to back at a thread-per-ray batch: the casts then do not
    trigger the next step's agent step early, so every step's gps / compass
    and the final state equal the serialised launches (nv_set_overlap 0)."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C3")
    W, H, n, steps = 256, 64, 512, 6
    suite = (nb.SensorConfig("depth", W, H), nb.SensorConfig("gps_compass"))
    sims = []
    for overlap in (0, 1):
        sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
        nat.check(sim.ctx.lib.nv_set_overlap(sim.ctx.handle, overlap))
        poses = synth.sample_poses(sc, n, seed=71)
        sim.reset(poses[:, :2], poses[:, 2])
        sims.append(sim)
    acts = torch.as_tensor(synth.random_actions(n, steps, seed=72), device="cuda:0")
    outs = []
    for k, sim in enumerate(sims):
        cam = sim.groups[0]["cam"]
        gps = torch.empty((steps, n, 2), dtype=torch.float64, device="cuda:0")
        comp = torch.empty((steps, n), dtype=torch.float64, device="cuda:0")
        st = nat.stream_handle()
        for s in range(steps):
            nat.check(sim.ctx.lib.nv_step_render(
                sim.ctx.handle, nat.ptr(acts[s]), cam, None, None, None, nat.ptr(gps[s]),
                nat.ptr(comp[s]), None, None, None, st))
            if k == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        outs.append((gps, comp, sim.state()))
    assert sims[1].ctx.faults() == 0
    (g0, c0, s0), (g1, c1, s1) = outs
    assert torch.equal(g0, g1)
    assert torch.equal(c0, c1)
    for a, b in zip(s0, s1):
        assert torch.equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("pinned", [False, True])
def test_host_steps_back_to_back_at_scale(nb, pinned):
    """Host-buffer steps issued back to back at the bench's batch size: each
    step's agent step and casts run beside the previous step's frame writer
    (alternating graphs, record halves and frame sets), and every step's host
    results and the final frames equal a serialised device-path replica."""
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C3")
    W, H, n, steps = 256, 256, 1024, 7
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("gps_compass"))
    a, b = (nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite,
                              floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
            for _ in range(2))
    poses = synth.sample_poses(sc, n, seed=61)
    for s in (a, b):
        s.reset(poses[:, :2], poses[:, 2])
    acts = synth.random_actions(n, steps, seed=62)
    if pinned:  # mapped host buffers: the kernels write the caller's arrays
        out = {"gps": torch.empty((n, 2), dtype=torch.float64).pin_memory(),
               "compass": torch.empty(n, dtype=torch.float64).pin_memory(),
               "collided": torch.empty(n, dtype=torch.uint8).pin_memory(),
               "displacement": torch.empty(n, dtype=torch.float64).pin_memory()}
    else:
        out = {"gps": np.empty((n, 2)), "compass": np.empty(n), "collided": np.empty(n, np.uint8),
               "displacement": np.empty(n)}
    got = []
    for t in range(steps):
        a.step_host(np.ascontiguousarray(acts[t]), out=out)
        got.append({k: (v.numpy() if hasattr(v, "numpy") else v).copy() for k, v in out.items()})
    for t in range(steps):
        b.step(torch.as_tensor(np.ascontiguousarray(acts[t]), device="cuda:0"))
        torch.cuda.synchronize()
        assert np.array_equal(got[t]["gps"], b.gps.cpu().numpy()), t
        assert np.array_equal(got[t]["compass"], b.compass.cpu().numpy()), t
        assert np.array_equal(got[t]["collided"], b.collided.cpu().numpy()), t
        assert np.array_equal(got[t]["displacement"], b.displacement.cpu().numpy()), t
    fr = a.host_step_frames()
    assert a.ctx.faults() == 0
    torch.cuda.synchronize()
    assert torch.equal(fr["rgb"], b.groups[0]["rgb"])
    assert torch.equal(fr["depth"], b.groups[0]["depth"])
    for x, y in zip(a.state(), b.state()):
        assert torch.equal(x, y)


def test_host_and_device_steps_share_a_side_stream(nb):
    """Host-buffer steps and device steps alternating on one non-default
    stream with no host synchronisation: a host step's frame writer still
    runs when the next device step's agent step and casts start, and each
    path has its own records, counters, pose records and ready flags, so
    every result equals a serialised device-path replica."""
    import ctypes
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C3")
    W, H, n, steps = 256, 128, 256, 8
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("gps_compass"))
    a, b = (nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite,
                              floor_color=sc.floor_color, ceiling_color=sc.ceiling_color)
            for _ in range(2))
    poses = synth.sample_poses(sc, n, seed=81)
    for s in (a, b):
        s.reset(poses[:, :2], poses[:, 2])
    acts = synth.random_actions(n, steps, seed=82)
    dacts = torch.as_tensor(acts, device="cuda:0")
    side = torch.cuda.Stream()
    sh = ctypes.c_void_p(side.cuda_stream)
    out = {"gps": torch.empty((n, 2), dtype=torch.float64).pin_memory(),
           "compass": torch.empty(n, dtype=torch.float64).pin_memory(),
           "collided": torch.empty(n, dtype=torch.uint8).pin_memory(),
           "displacement": torch.empty(n, dtype=torch.float64).pin_memory()}
    torch.cuda.synchronize()
    got = {}
    for t in range(steps):
        if t % 2 == 0:
            a.step_host(np.ascontiguousarray(acts[t]), out=out, stream=sh)
            got[t] = out["gps"].numpy().copy()
        else:
            a.step(dacts[t], stream=sh)
    side.synchronize()
    for t in range(steps):
        b.step(dacts[t])
        torch.cuda.synchronize()
        if t in got:
            assert np.array_equal(got[t], b.gps.cpu().numpy()), t
    torch.cuda.synchronize()
    assert a.ctx.faults() == 0
    assert torch.equal(a.groups[0]["rgb"], b.groups[0]["rgb"])
    assert torch.equal(a.groups[0]["depth"], b.groups[0]["depth"])
    assert torch.equal(a.gps, b.gps)
    for x, y in zip(a.state(), b.state()):
        assert torch.equal(x, y)


def test_host_buffer_path_matches_device_path(nb):
    """nv_step_render_host (graph-replayed, packed results) gives the same step
    results as nv_step_render on device buffers, across repeated
    calls (graph replay), a camera/channel change (re-capture) and a fill-mode
    change (generation bump)."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C2")
    W, H, n = 128, 64, 40
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("gps_compass"))
    sims = [nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
            for _ in range(2)]
    poses = synth.sample_poses(sc, n, seed=31)
    for s in sims:
        s.reset(poses[:, :2], poses[:, 2])
    acts = synth.random_actions(n, 8, seed=32)
    out = {"gps": np.empty((n, 2)), "compass": np.empty(n), "collided": np.empty(n, np.uint8),
           "displacement": np.empty(n)}
    for t in range(acts.shape[0]):
        if t == 5:
            for s in sims:
                nat.check(s.ctx.lib.nv_set_fill_mode(s.ctx.handle, nat.NV_FILL_GENERIC))
        a_host = np.ascontiguousarray(acts[t])
        sims[0].step_host(a_host, out=out)
        sims[1].step(torch.as_tensor(a_host, device="cuda:0"))
        torch.cuda.synchronize()
        o1 = sims[1].observations()
        assert np.array_equal(out["gps"], o1["gps"].cpu().numpy())
        assert np.array_equal(out["compass"], o1["compass"].cpu().numpy())
        assert np.array_equal(out["collided"], sims[1].collided.cpu().numpy())
        assert np.array_equal(out["displacement"], sims[1].displacement.cpu().numpy())
    # pinned (mapped) output buffers: the kernels write them directly
    pin = {"gps": torch.empty((n, 2), dtype=torch.float64).pin_memory(),
           "compass": torch.empty(n, dtype=torch.float64).pin_memory(),
           "collided": torch.empty(n, dtype=torch.uint8).pin_memory(),
           "displacement": torch.empty(n, dtype=torch.float64).pin_memory()}
    for t in range(3):
        a_host = np.ascontiguousarray(acts[t])
        sims[0].step_host(a_host, out=pin)
        sims[1].step(torch.as_tensor(a_host, device="cuda:0"))
        torch.cuda.synchronize()
        assert torch.equal(pin["gps"], sims[1].gps.cpu())
        assert torch.equal(pin["compass"], sims[1].compass.cpu())
        assert torch.equal(pin["collided"], sims[1].collided.cpu())
        assert torch.equal(pin["displacement"], sims[1].displacement.cpu())
    # the non-graph path (host frames requested) agrees too
    a_host = np.ascontiguousarray(acts[0])
    rgb_h = np.empty((n, H, W, 3), np.uint8)
    out["rgb"] = rgb_h
    sims[0].step_host(a_host, out=out, frames_to_host=True)
    sims[1].step(torch.as_tensor(a_host, device="cuda:0"))
    torch.cuda.synchronize()
    assert np.array_equal(rgb_h, sims[1].observations()["rgb"].cpu().numpy())
    assert np.array_equal(out["gps"], sims[1].gps.cpu().numpy())


@pytest.mark.parametrize("mode", ["plain", "no-overlap", "thread", "warp"])
def test_host_buffer_path_first_call_all_modes(nb, mode):
    """The host-buffer step as the very first call on a fresh simulator (its
    graph is captured before any device step ran: every lazily allocated
    buffer must exist before the capture) in each step-launch mode, against
    the device-buffer path."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C2")
    W, H, n = 128, 64, 200  # 25,600 rays: the thread-per-ray cast
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("gps_compass"))
    sims = [nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
            for _ in range(2)]
    poses = synth.sample_poses(sc, n, seed=41)
    for s in sims:
        s.reset(poses[:, :2], poses[:, 2])
        c = s.ctx
        if mode == "no-overlap":
            nat.check(c.lib.nv_set_overlap(c.handle, 0))
        elif mode == "thread":
            nat.check(c.lib.nv_set_cast_mode(c.handle, nat.NV_CAST_THREAD))
        elif mode == "warp":
            nat.check(c.lib.nv_set_cast_mode(c.handle, nat.NV_CAST_WARP))
    acts = synth.random_actions(n, 4, seed=42)
    out = {"gps": np.empty((n, 2)), "compass": np.empty(n), "collided": np.empty(n, np.uint8),
           "displacement": np.empty(n)}
    for t in range(acts.shape[0]):
        a_host = np.ascontiguousarray(acts[t])
        sims[0].step_host(a_host, out=out)
        sims[1].step(torch.as_tensor(a_host, device="cuda:0"))
        torch.cuda.synchronize()
        assert np.array_equal(out["gps"], sims[1].gps.cpu().numpy())
        assert np.array_equal(out["collided"], sims[1].collided.cpu().numpy())
        assert np.array_equal(out["displacement"], sims[1].displacement.cpu().numpy())


def test_host_step_frames_and_interleaving(nb):
    """A host-buffer step returns once its step results are in (its frame
    writer may still run): nv_host_frames waits for the frames, and device
    steps interleaved on the same context keep every result and frame equal
    to a pure device-path replica."""
    import ctypes
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth

    class _Dev:  # zero-copy torch view of a device pointer
        def __init__(self, ptr, shape, typestr):
            self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr,
                                             "data": (ptr, False), "version": 3}

    sc = synth.config_scene("C2")
    W, H, n = 128, 64, 200
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("gps_compass"))
    a, b = (nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
            for _ in range(2))
    poses = synth.sample_poses(sc, n, seed=51)
    for s in (a, b):
        s.reset(poses[:, :2], poses[:, 2])
    acts = synth.random_actions(n, 8, seed=52)
    out = {"gps": np.empty((n, 2)), "compass": np.empty(n), "collided": np.empty(n, np.uint8),
           "displacement": np.empty(n)}
    for t in range(acts.shape[0]):
        a_host = np.ascontiguousarray(acts[t])
        b.step(torch.as_tensor(a_host, device="cuda:0"))
        if t % 3 != 2:
            a.step_host(a_host, out=out)
            rgb_p, dep_p = ctypes.c_void_p(), ctypes.c_void_p()
            nat.check(a.ctx.lib.nv_host_frames(a.ctx.handle, 0, ctypes.byref(rgb_p),
                                               ctypes.byref(dep_p), None))
            rgb = torch.as_tensor(_Dev(rgb_p.value, (n, H, W, 3), "|u1"), device="cuda:0")
            dep = torch.as_tensor(_Dev(dep_p.value, (n, H, W), "<f4"), device="cuda:0")
            gps = out["gps"]
        else:
            a.step(torch.as_tensor(a_host, device="cuda:0"))
            rgb, dep = a.groups[0]["rgb"], a.groups[0]["depth"]
            gps = a.gps.cpu().numpy()
        torch.cuda.synchronize()
        assert np.array_equal(gps, b.gps.cpu().numpy()), t
        assert torch.equal(rgb, b.groups[0]["rgb"]), t
        assert torch.equal(dep, b.groups[0]["depth"]), t
