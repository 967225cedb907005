"""bench.py's JSON contract: the reference (oracle) arm on CPU, our arm on the GPU."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["unit"] == "GLUPS" and d["value"] > 0
    assert d["config"]["workload"] == "C1" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert {"cpu_model", "nproc", "pinned_core"} <= set(d["cpu_baseline"])
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["gpu_launches"] == 0


def test_gpus_flag_refuses_missing_devices():
    """--gpus N outside torchrun re-launches under torch.distributed.run, or exits non-zero
    when fewer than N devices are visible (this container has none)."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:
        have = 0
    if have < 2:
        assert p.returncode != 0 and "only %d CUDA device" % have in p.stderr


@pytest.mark.gpu
def test_gpu_arm_line_has_every_key():
    d = run_bench("--config", "C2", "--steps", "2", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches",
              "other_mode"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["dtype"] == "f64" and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["workload"] == "C2" and d["config"]["mode"] == "matched"
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] <= 1.0
    assert d["other_mode"]["mode"] == "fast" and d["other_mode"]["value"] > 0
    assert d["other_mode"]["roofline"]["reduced_op_form"] is True
    assert d["parity_check"]["ok"] is True and d["parity_check"]["criterion"] == "bitwise"
    assert len(d["step_stats"]["ms_all"]) == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    e = d["e2e"]
    assert set(e["variants"]) == {"solve_host", "set_initial+run+get"}
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * 1_000_000 == e["d2h_bytes_per_step"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
