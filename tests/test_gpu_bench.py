"""bench.py on the GPU (small runs): the JSON contract of the single-rank line, and the
multi-rank control flow (`--gpus 2` self-launch; RAAS_BENCH_SHARE_GPU=1 lets both ranks share the
box's one GPU over gloo: a functional check, never a measurement) for request sharding (weak and
strong scaling) and head sharding."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, share=False, timeout=900):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    if share:
        env["RAAS_BENCH_SHARE_GPU"] = "1"
    r = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout, env=env)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0]), r.stderr


def test_single_rank_line_contract():
    d, _ = _bench(["--config", "2", "--layers", "4", "--steps", "20", "--warmup", "3",
                   "--cpu-seconds", "2"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["unit"] == "decode steps/s" and d["value"] > 0
    assert d["gpu_launches"] == 20 * 4 and d["device_status"] == 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.3
    assert d["e2e"]["unit"] == d["unit"] and d["e2e"]["h2d_bytes_per_step"] > 0
    # config 2 caches are rotated to >= 4x L2 of distinct K/V (SURVEY §8(d) L2 hygiene)
    assert ">= 4x L2" in d["config"]["l2"]


@pytest.mark.parametrize("extra,mode", [
    (["--config", "3", "--batch", "8", "--layers", "2"], "weak"),
    (["--config", "4", "--scaling", "strong", "--batch", "16", "--layers", "2"], "strong"),
    (["--config", "2", "--shard", "heads", "--layers", "2"], "heads"),
])
def test_two_ranks_self_launched_share_gpu(extra, mode):
    """`python bench.py --gpus 2`: two ranks, both busy (per-rank device times > 0), one line
    with n_gpus = 2 and the max over ranks as the step time."""
    d, err = _bench(["--gpus", "2", "--steps", "6", "--warmup", "3", "--no-e2e"] + extra, share=True)
    assert d["n_gpus"] == 2 and "not a measurement" in d["note"]
    assert len(d["per_rank_ms"]) == 2 and min(d["per_rank_ms"]) > 0
    assert abs(d["ms_per_step"] * 6 - max(d["per_rank_ms"])) < 1e-6 * max(d["per_rank_ms"]) + 1e-9
    assert d["scaling"] == ("weak" if mode == "weak" else "strong")
    if mode == "strong":
        assert d["config"]["global_batch"] == 16 and d["config"]["per_gpu_batch"] == 8
    if mode == "heads":
        assert "head-sharded x2" in d["config"]["parallelism"]
    assert "[rank 0]" in err and "[rank 1]" in err
