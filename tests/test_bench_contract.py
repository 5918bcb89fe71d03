"""bench.py's reference arm runs on the CPU (the oracle port) and prints the
contract's JSON line -- checked here without a GPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--ref-seconds", "1"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["warmup"] >= 3
    assert line["cpu_baseline"]["kind"] in ("port", "reference")
    assert line["cpu_baseline"]["cores"] >= 1 and line["cpu_baseline"]["sample"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"]


def _line(args, timeout=600):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_reference_arm_reports_the_workload_config():
    """The reference arm prints the GPU arm's workload config (same dict:
    envs, resolution, channels, scene size, parallelism, scaling) and how
    many envs its bounded sample stepped."""
    line = _line(["--impl", "reference", "--steps", "1", "--warmup", "3", "--ref-seconds", "1"])
    cfg = line["config"]
    assert cfg["envs_per_gpu"] == 1024 and cfg["envs_total"] == 1024
    assert (cfg["width"], cfg["height"], cfg["channels"]) == (256, 256, ["rgb", "depth"])
    assert cfg["segments"] > 90_000 and cfg["scaling"] == "weak"
    assert 1 <= line["sampled_envs"] <= 1024


def test_bench_spawns_its_own_ranks_dry_run():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks itself (one
    process per GPU); with the GPU parts stubbed (gloo on CPU) rank 0 prints
    n_gpus = 2 and the all-gathered per-env records arrive in global env
    order."""
    line = _line(["--gpus", "2", "--dry-run", "--steps", "2"])
    assert line["n_gpus"] == 2 and line["dry_run"] is True
    assert line["config"]["envs_total"] == 2048 and line["config"]["envs_per_gpu"] == 1024
    assert line["gathered_records"] == 2048 and line["gathered_in_env_order"] is True


def test_bench_strong_scaling_preset_dry_run():
    """--scaling strong: the config's 1024 envs in total, split over the GPUs."""
    line = _line(["--gpus", "4", "--dry-run", "--scaling", "strong", "--steps", "2"])
    assert line["n_gpus"] == 4 and line["scaling"] == "strong"
    assert line["config"]["envs_total"] == 1024 and line["config"]["envs_per_gpu"] == 256
    assert line["gathered_records"] == 1024 and line["gathered_in_env_order"] is True


def test_bench_rank_count_mismatch_is_an_error():
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300,
                         env=dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"))
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr
