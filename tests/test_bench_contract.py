"""The bench.py JSON-line contract the driver reads (a short run at r = 64 so the
test stays quick): one JSON line with the required keys, a measured e2e figure
with its host<->device bytes, the roofline block, the clocks sample, a positive
launch count, and the lane trial of the warm-up."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_json_line_contract():
    out = subprocess.run([sys.executable, "bench.py", "--steps", "4", "--warmup", "3", "--r", "64",
                          "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] < 1 and rf["bound"] == "hbm" and rf["unit"] == "GB/s"
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    sel = d["config"]["lane_selection"]
    assert sel["chosen"] in (1, 2) and sel["wall_s_1_lanes"] > 0 and sel["wall_s_2_lanes"] > 0
    assert d["config"]["designs_in_flight_per_gpu"] == sel["chosen"]
