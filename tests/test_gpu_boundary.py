"""Drop-in boundary behaviours of the C ABI and its facades (round-2 fixes):

* Simulator.observations() before set_agent_state renders the reference's
  initial AgentState (origin, heading 0; sim.py:159, 192-200);
* nv_step_render_host renders every camera group (NV_ALL_CAMERAS), not only
  the first;
* the host-step graph is re-captured when a buffer it uses is reallocated
  (never replayed into freed memory).
"""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

POSE_ATOL = 1e-6


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_01201_b200 as nb
    from paper_1904_01201_b200 import _native
    _native.load()
    return nb


def _square(nb):
    walls = [nb.WallSegment(a=(0.0, 0.0), b=(10.0, 0.0), semantic_id=1, albedo=(0.6, 0.5, 0.4)),
             nb.WallSegment(a=(10.0, 0.0), b=(10.0, 10.0), semantic_id=2, albedo=(0.5, 0.6, 0.4)),
             nb.WallSegment(a=(10.0, 10.0), b=(0.0, 10.0), semantic_id=3, albedo=(0.4, 0.5, 0.6)),
             nb.WallSegment(a=(0.0, 10.0), b=(0.0, 0.0), semantic_id=4, albedo=(0.6, 0.4, 0.5)),
             nb.WallSegment(a=(-3.0, -2.0), b=(-3.0, 2.0), semantic_id=5, albedo=(0.2, 0.9, 0.3))]
    return nb.Scene(id="square-10", walls=walls, floor_color=(0.3, 0.3, 0.3),
                    ceiling_color=(0.9, 0.9, 0.9), wall_height=2.5)


def test_observations_before_reset_render_initial_state(nb, oracle_mod):
    """The reference renders at AgentState(position=0, heading=0) when
    observations() is called before set_agent_state (sim.py:159, 192-200);
    with a gps_compass sensor it fails in gps_compass(state, None)."""
    scene = _square(nb)
    graph = nb.build_scene_graph(scene)
    W, H = 64, 48
    cfgs = (nb.SensorConfig("rgb", width=W, height=H), nb.SensorConfig("depth", width=W, height=H),
            nb.SensorConfig("semantic", width=W, height=H))
    sim = nb.Simulator(graph, sensor_configs=cfgs)
    obs = sim.observations()
    segs, sem, alb = nb.flatten_arrays(graph)
    osc = oracle_mod.OracleScene(segs, sem, alb, scene.wall_height, scene.floor_color,
                                 scene.ceiling_color)
    rgb, dep, sm = osc.render((0.0, 0.0), 0.0, 1.5, W, H, focal=cfgs[0].focal)
    assert np.array_equal(obs.semantic, sm)
    assert np.all(np.abs(obs.depth - dep) <= 1e-5 * np.maximum(dep, 1e-9))
    assert np.max(np.abs(obs.rgb - rgb)) <= 1.0 / 255 + 1e-9
    assert (obs.semantic != 0).any()  # from the room's corner: walls in view
    sim_g = nb.Simulator(graph, sensor_configs=cfgs + (nb.SensorConfig("gps_compass"),))
    with pytest.raises(AttributeError):
        sim_g.observations()
    sim_g.set_agent_state((5.0, 5.0), 0.3)
    o2 = sim_g.observations()
    assert np.allclose(o2.gps, [0.0, 0.0], atol=1e-12)


def test_step_host_renders_every_camera_group(nb):
    """A suite with two resolutions: the host-buffer step renders both camera
    groups (NV_ALL_CAMERAS) with the same frames and step results as the
    device path."""
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C2")
    n = 24
    suite = (nb.SensorConfig("rgb", 128, 64), nb.SensorConfig("depth", 64, 48),
             nb.SensorConfig("semantic", 64, 48), nb.SensorConfig("gps_compass"))
    sims = [nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
            for _ in range(2)]
    assert len(sims[0].groups) == 2
    poses = synth.sample_poses(sc, n, seed=61)
    for s in sims:
        s.reset(poses[:, :2], poses[:, 2])
    acts = synth.random_actions(n, 6, seed=62)
    out = {"gps": np.empty((n, 2)), "compass": np.empty(n), "collided": np.empty(n, np.uint8),
           "displacement": np.empty(n)}
    for t in range(acts.shape[0]):
        a_host = np.ascontiguousarray(acts[t])
        sims[0].step_host(a_host, out=out)
        sims[1].step(torch.as_tensor(a_host, device="cuda:0"))
        torch.cuda.synchronize()
        fr = sims[0].host_step_frames()
        dev = sims[1].observations()
        assert set(fr) == {"rgb", "depth", "semantic"}
        assert torch.equal(fr["rgb"], dev["rgb"]), t
        assert torch.equal(fr["depth"], dev["depth"]), t
        assert torch.equal(fr["semantic"].view(torch.int16), dev["semantic"].view(torch.int16)), t
        assert np.array_equal(out["gps"], sims[1].gps.cpu().numpy())
        assert np.array_equal(out["collided"], sims[1].collided.cpu().numpy())
    with pytest.raises(nb.SensorError):
        sims[0].step_host(np.ascontiguousarray(acts[0]), out=dict(out), frames_to_host=True)


def test_host_step_graph_recaptured_after_buffer_growth(nb):
    """nv_fill_frames with more frames than envs grows the camera's record
    buffer; the next host-buffer step must not replay its cached graph into
    the freed buffer (it re-captures) and still matches the device path."""
    from paper_1904_01201_b200 import _native as nat
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C2")
    W, H, n = 128, 64, 16
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("gps_compass"))
    sims = [nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
            for _ in range(2)]
    poses = synth.sample_poses(sc, n, seed=71)
    for s in sims:
        s.reset(poses[:, :2], poses[:, 2])
    acts = synth.random_actions(n, 6, seed=72)
    out = {"gps": np.empty((n, 2)), "compass": np.empty(n), "collided": np.empty(n, np.uint8),
           "displacement": np.empty(n)}
    c = sims[0].ctx
    for t in range(acts.shape[0]):
        if t == 3:  # grow the record buffer through the operator entry
            m = 8 * n
            tc = torch.full((m, W), float("inf"), dtype=torch.float64, device="cuda:0")
            ic = torch.full((m, W), -1, dtype=torch.int64, device="cuda:0")
            dx = torch.ones((m, W), dtype=torch.float64, device="cuda:0")
            dy = torch.zeros((m, W), dtype=torch.float64, device="cuda:0")
            dep = torch.empty((m, H, W), dtype=torch.float32, device="cuda:0")
            nat.check(c.lib.nv_fill_frames(c.handle, 0, m, nat.ptr(tc), nat.ptr(ic), nat.ptr(dx),
                                           nat.ptr(dy), 1.5, None, nat.ptr(dep), None,
                                           nat.stream_handle("cuda:0")))
            torch.cuda.synchronize()
            assert bool((dep <= 10.0).all())  # every column missed: floor / ceiling / void
        a_host = np.ascontiguousarray(acts[t])
        sims[0].step_host(a_host, out=out)
        sims[1].step(torch.as_tensor(a_host, device="cuda:0"))
        torch.cuda.synchronize()
        fr = sims[0].host_step_frames()
        assert torch.equal(fr["rgb"], sims[1].observations()["rgb"]), t
        assert torch.equal(fr["depth"], sims[1].observations()["depth"]), t
        assert np.array_equal(out["gps"], sims[1].gps.cpu().numpy())
