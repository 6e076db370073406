"""CPU checks of bench.py's control flow: the reference arm (`--impl reference`, the fp64 oracle
on host cores) prints one JSON line with the contract's keys, on the metric and unit of the GPU
arm (byte-identical, so the driver can compute the ratio); `--gpus 2` without torchrun launches
two ranks itself (gloo for the CPU-only reference arm) and still prints exactly one line."""
import importlib.util
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench_module():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    r = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True, text=True,
                       timeout=300, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def _check_reference_line(d, bench, n_gpus):
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is True
    # the GPU arm prints the same metric and unit strings (bench.METRIC / bench.UNIT)
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["n_gpus"] == n_gpus
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"] == bench.CONFIGS[1]["workload"]


def test_reference_arm_json_line():
    bench = _bench_module()
    d = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "3",
              "--cpu-seconds", "1"])
    _check_reference_line(d, bench, 1)


def test_reference_arm_two_ranks_self_launched():
    """`python bench.py --gpus 2` (no torchrun): bench.py spawns rank 0 and rank 1 with the
    torchrun environment, they rendezvous (gloo, 127.0.0.1), rank 0 alone measures and prints
    one line with n_gpus = 2, rank 1 exits 0 after the barriers."""
    bench = _bench_module()
    d = _run(["--impl", "reference", "--gpus", "2", "--config", "1", "--steps", "1", "--warmup",
              "3", "--cpu-seconds", "1"])
    _check_reference_line(d, bench, 2)


def test_gpus_must_match_world_size_under_torchrun():
    e = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--config", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=120, env=e)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_unit_detail_and_rotation_helpers():
    bench = _bench_module()
    assert "summed over 2 GPU" in bench.unit_detail(64, 32, 2, "weak")
    assert "global batch (256 requests over 8 GPUs)" in bench.unit_detail(256, 28, 8, "strong")
    l2 = 126 * 2**20
    # config 2: 32 layers x 8 units x 64 pages x 8 KiB = 128 MiB per model step -> 4 rotations
    assert bench.l2_rotation(32 * 8 * 64 * 8192, l2) == 4
    assert bench.l2_rotation(16 * 2**30, l2) == 1          # config 3: 16 GiB
    assert bench.l2_rotation(32 * 1024, l2) == 64          # toy: capped
