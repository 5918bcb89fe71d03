"""The nav/task oracle (oracle/navsim_nav_oracle.c) against fixtures produced
by the unmodified reference (tests/golden/make_golden_task.py): occupancy
masks, clearances, goal snapping, distance fields and geodesic queries
bit-exact, and whole PointGoal episodes (per-step distance, reward, done,
kinematics, final EpisodeOutcome) bit-exact."""
import glob
import os

import numpy as np
import pytest

from oracle import nav_oracle as no
from oracle import oracle as orc

HERE = os.path.dirname(os.path.abspath(__file__))
FILES = sorted(glob.glob(os.path.join(HERE, "golden", "golden_task_*.npz")))


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module", params=FILES, ids=[os.path.basename(f)[12:-4] for f in FILES])
def gold(request):
    return np.load(request.param)


def test_mask_clearance_exact(gold):
    segs, bnds = gold["segments"], tuple(gold["bounds"])
    for key in [k[:-7] for k in gold.files if k.endswith("_origin")]:
        r = int(key[1:]) / 1000.0
        g = no.Grid(segs, bnds, 0.05, r)
        assert np.array_equal(g.origin, gold[f"{key}_origin"])
        assert np.array_equal(g.navigable, gold[f"{key}_navigable"]), key
        assert np.array_equal(g.clearance.ravel()[gold[f"{key}_clearance_idx"]],
                              gold[f"{key}_clearance_val"])
        assert sha(g.clearance) == str(gold[f"{key}_clearance_sha"])


def test_snap_fields_geodesic_exact(gold):
    g = no.Grid(gold["segments"], tuple(gold["bounds"]))
    for p, c in zip(gold["snap_pts"], gold["snap_cells"]):
        got = g.snap(p)
        assert (got if got is not None else (-1, -1)) == tuple(c)
    for k, goal in enumerate(gold["field_goal"]):
        cell = g.snap(goal)
        assert cell == tuple(gold["field_cell"][k])
        f = g.field(cell)
        assert np.array_equal(f.ravel()[gold["field_idx"][k]], gold["field_val"][k])
        assert sha(f) == str(gold["field_sha"][k])
        for p, v in zip(gold["geo_pts"][k], gold["geo_val"][k]):
            if np.isnan(v):
                with pytest.raises(ValueError):
                    g.geodesic(f, p)
            else:
                got = g.geodesic(f, p)
                assert got == v or (np.isinf(got) and np.isinf(v))


def test_episodes_exact(gold):
    if "n_episodes" not in gold.files:
        pytest.skip("no episodes in this fixture")
    segs = gold["segments"]
    n = len(segs)
    scene = orc.OracleScene(segs, np.arange(1, n + 1), np.full((n, 3), 0.5))
    env = no.TaskEnv(scene, no.Grid(segs, tuple(gold["bounds"])))
    for k in range(int(gold["n_episodes"])):
        p = f"ep{k}_"
        sr = gold[p + "start_raw"]
        d0 = env.reset(sr[:2], sr[2], gold[p + "goal"], float(gold[p + "gdsp"]))
        assert d0 == float(gold[p + "d0"])
        assert env.state[:3] == list(gold[p + "start"])
        out = None
        for a, row in zip(gold[p + "actions"], gold[p + "rows"]):
            d, r, done, coll, moved, out = env.step(int(a))
            assert (d, r, float(done), float(coll), moved) == tuple(row[:5])
            assert env.state[:3] == list(row[5:8])
        o = gold[p + "outcome"]
        assert out is not None
        assert (float(out["success"]), float(out["path_taken"]), out["spl"], float(out["steps"]),
                float(out["collisions"]), float(out["terminated_by"])) == \
            (o[0], o[2], o[3], o[4], o[5], o[6])
