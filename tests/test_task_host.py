"""Host-side task arithmetic mirrors (task.py:91-115 restated in
paper_1904_01201_b200.task), checked like the reference's
pkg/tests/test_task.py:16-60 / :172 -- no GPU needed.  The device versions
of the same arithmetic are checked bit-exact against the oracle in
test_gpu_task.py."""
import math

import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

lengths = st.floats(min_value=1e-3, max_value=1e4, allow_nan=False)


@pytest.fixture(scope="module")
def task():
    from paper_1904_01201_b200 import task
    return task


def test_spl_point_values(task):  # test_task.py:16
    assert task.spl(True, 10.0, 10.0) == 1.0
    assert task.spl(True, 5.0, 10.0) == 0.5
    assert task.spl(False, 3.0, 100.0) == 0.0


@given(st.booleans(), lengths, lengths)
def test_spl_algebra(success, shortest, taken):  # test_task.py:23
    from paper_1904_01201_b200.task import spl
    v = spl(success, shortest, taken)
    assert 0.0 <= v <= (1.0 if success else 0.0)
    if success:
        assert (v == 1.0) == (taken <= shortest)
        assert spl(success, shortest, taken * 2) <= v


def test_spl_rejects_bad_lengths(task):  # test_task.py:32
    with pytest.raises(task.TaskError):
        task.spl(True, 0.0, 1.0)
    with pytest.raises(task.TaskError):
        task.spl(True, 1.0, -1.0)


def test_reward_point_values_and_telescoping(task):  # test_task.py:39, :46
    assert task.reward(0.5, 0.1, True) == pytest.approx(10.39, abs=1e-12)
    assert task.reward(1.0, 1.0, False) == pytest.approx(-0.01, abs=1e-15)
    custom = task.RewardParams(success_reward=2.0, step_penalty=-0.5)
    assert task.reward(1.0, 0.5, True, custom) == pytest.approx(2.0, abs=1e-12)
    d = np.abs(np.random.default_rng(2).normal(5.0, 2.0, size=51))
    total = sum(task.reward(d[k], d[k + 1], False) for k in range(50))
    assert total == pytest.approx(d[0] - d[50] + 50 * (-0.01), abs=1e-9)


def test_success_boundary(task):  # test_task.py:55
    assert task.success_test(0.0)
    assert task.success_test(0.2)
    assert not task.success_test(0.2 + 1e-12)


def test_outcome_json_roundtrip(task):  # test_task.py:172
    out = task.EpisodeOutcome(success=True, shortest_path=5.0, path_taken=6.0, spl=5.0 / 6.0,
                              steps=30, collisions=2, terminated_by="stop")
    assert task.EpisodeOutcome.from_json(out.to_json()) == out
