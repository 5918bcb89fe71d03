"""Pin the C oracle to the reference: every golden array produced by the
unmodified navsim (tests/golden/make_golden.py) must be reproduced bit-exactly."""
import hashlib

import numpy as np
import pytest

from conftest import golden_names, load_golden

NAMES = golden_names()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module", params=NAMES)
def case(request, oracle_mod):
    g = load_golden(request.param)
    sc = oracle_mod.OracleScene(g["segments"], g["semantic_ids"], g["albedo"],
                                float(g["wall_height"]), g["floor_color"], g["ceiling_color"])
    return request.param, g, sc


def test_goldens_present():
    assert len(NAMES) >= 6


def test_grid_build(case):
    _, g, sc = case
    x0, y0, nx, ny, starts, items = sc.grid()
    assert (x0, y0, nx, ny) == (g["grid_x0"], g["grid_y0"], g["grid_nx"], g["grid_ny"])
    assert np.array_equal(starts, g["grid_starts"])
    assert np.array_equal(items, g["grid_items"])


def test_column_directions(case, oracle_mod):
    _, g, _ = case
    for k, (_, _, h) in enumerate(g["poses"]):
        dx, dy = oracle_mod.column_directions(h, 256, float(g["cast_focal"]))
        assert np.array_equal(dx, g["cast_dirs"][k][:, 0])
        assert np.array_equal(dy, g["cast_dirs"][k][:, 1])


def test_raycasts_bit_exact(case):
    _, g, sc = case
    for k, (x, y, _) in enumerate(g["poses"]):
        t, i = sc.raycast((x, y), g["cast_dirs"][k])
        assert np.array_equal(i, g["cast_i_grid"][k])
        assert np.array_equal(t, g["cast_t_grid"][k])
        t, i = sc.raycast((x, y), g["cast_dirs"][k], brute=True)
        assert np.array_equal(i, g["cast_i_brute"][k])
        assert np.array_equal(t, g["cast_t_brute"][k])


def test_frames_bit_exact(case):
    _, g, sc = case
    keys = sorted(k[:-len("_focal")] for k in g if k.startswith("frame_") and k.endswith("_focal"))
    assert keys
    for key in keys:
        w, h = (int(v) for v in key[len("frame_"):].split("x"))
        for k, (x, y, hd) in enumerate(g["poses"]):
            rgb, dep, sem = sc.render((x, y), hd, float(g["sensor_height"]), width=w, height=h)
            assert sha(rgb) == g[key + "_rgb_sha"][k]
            assert sha(dep) == g[key + "_depth_sha"][k]
            assert np.array_equal(sem, g[key + "_sem"][k])


def test_kinematics_bit_exact(case, oracle_mod):
    _, g, sc = case
    for e, (x, y, h) in enumerate(g["kin_starts"]):
        st = [x, y, oracle_mod.wrap_angle(h), 0.0, 0]
        for s, a in enumerate(g["kin_actions"][e]):
            st, collided, moved = sc.step(st, int(a))
            assert st[:4] == list(g["kin_states"][e][s][:4]), (e, s)
            assert st[4] == g["kin_states"][e][s][4]
            assert collided == bool(g["kin_collided"][e][s])
            assert moved == g["kin_moved"][e][s]


def test_disc_cast_and_clearance(case):
    _, g, sc = case
    for q, res, clr in zip(g["disc_queries"], g["disc_results"], g["clearance"]):
        t, i, tan = sc.cast_disc(q[:2], q[2:4], q[4])
        got = np.array([t, float(i), tan[0], tan[1]])
        assert np.array_equal(got, res)
        assert sc.clearance(q[:2]) == clr
