"""CPU: bench.py's reference arm (the driver runs `bench.py --impl reference` on
the GPU box at round end) end to end on a small CPU sample, for the N = 1
(cfg2 subtree) and N > 1 (cfg3 family) workloads, and the JSON contract keys."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _ref_available():
    from oracle import ref_driver as rd

    return rd.AVAILABLE


@pytest.mark.skipif(not _ref_available(), reason="reference package not importable here")
@pytest.mark.parametrize("extra,workload", [([], "cfg2"), (["--gpus", "2"], "cfg3")])
def test_reference_arm_line(extra, workload):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup",
                          "0", "--cpu-sample-rows", "1024"] + extra, capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "reference"
    assert line["config"]["rank"] == (32 if workload == "cfg2" else 64)
    assert line["e2e"]["h2d_bytes_per_step"] == 0
