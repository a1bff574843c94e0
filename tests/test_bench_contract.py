"""bench.py keeps the driver's JSON-line contract: the reference arm (the fp64 oracle on the
host cores) on CPU, and the GPU arm on a small batch (-m gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         cwd=ROOT, timeout=timeout)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-sample-events", "1"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "pairs/s" and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and "sample" in cb
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_gpu_arm_json_line():
    d = _run(["--events", "40", "--steps", "5", "--warmup", "3", "--cpu-plan", "quick", "--e2e-steps", "1"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["scaling"] == "strong"
    assert d["config"]["events_total"] == 40 and d["gathered"]["ranks"] == [0]
    assert d["gathered"]["event_base"] == [0] and d["per_rank"][0]["events"] == 40
    assert all(len(v) == 5 for v in d["phases_ms_per_step_all_steps"].values())
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["dtype"] == "f32" and d["data"] == "synthetic"
    r = d["roofline"]
    assert r["bound"] in ("alu", "tensor", "hbm") and 0 < r["frac"] <= 1.0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and "traffic" in r
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["cpu_model"]
    assert cb["all_cores"]["threads"] == cb["cores"] and cb["one_core"]["threads"] == 1
    assert d["config"]["workload"].startswith("cfg3")


def test_gpus_n_spawns_ranks_and_shards_the_batch():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks itself (torch.distributed.run on
    127.0.0.1); each rank takes its contiguous block of the SAME batch (strong scaling, SURVEY.md
    §8(e)).  --dist-check does no GPU work: gloo all_gather of the shard bounds and hit counts."""
    from synth import configs as C
    from synth import events as G
    d = _run(["--gpus", "2", "--dist-check", "--config", "cfg2"], timeout=900)
    assert d["world"] == 2 and d["scaling"] == "strong"
    sh = sorted(d["shards"])
    assert [s[0] for s in sh] == [0, 1] and sh[0][1] == 0 and sh[0][2] == sh[1][1] and sh[1][2] == 200
    full = G.make_batch(C.CFG2, range(200))
    assert sum(s[3] for s in sh) == full.n_hits
    w = _run(["--gpus", "2", "--dist-check", "--config", "cfg2", "--scaling", "weak", "--events-per-rank", "7"],
             timeout=900)
    assert sorted(s[1:3] for s in w["shards"]) == [[0, 7], [7, 14]] and w["scaling"] == "weak"
    r = _run(["--gpus", "2", "--dist-check", "--config", "cfg1"], timeout=900)
    assert r["scaling"] == "replicas" and all(s[1:3] == [0, 1] for s in r["shards"])
