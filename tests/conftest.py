import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

# achieved parity errors, reported at the end of the session (and written to
# gpurun_out/parity_errors.json on a GPU box) -- the gates are in the tests
PARITY_LOG: list = []


def record_parity(case: str, **errs) -> None:
    """Log one case's achieved errors (relative, vs the oracle / reference) and gates."""
    PARITY_LOG.append({"case": case, **{k: (float(v) if v is not None else None) for k, v in errs.items()}})


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device and the built native library")


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if not PARITY_LOG:
        return
    tr = terminalreporter
    tr.write_sep("-", f"achieved parity errors ({len(PARITY_LOG)} cases)")
    for row in PARITY_LOG:
        tr.write_line(row["case"] + "  " + "  ".join(f"{k}={v:.2e}" for k, v in row.items()
                                                     if k != "case" and v is not None))
    out = ROOT / "gpurun_out"
    if out.is_dir() and os.environ.get("HODLR_PARITY_JSON", "1") == "1":
        (out / "parity_errors.json").write_text(json.dumps(PARITY_LOG, indent=1))
