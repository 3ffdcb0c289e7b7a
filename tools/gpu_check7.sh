mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3w_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s3w_pytest.log; grep -E "FAIL|Error|assert" gpurun_out/s3w_pytest.log | head -5
timeout 300 python tools/cfg5_ab.py 1 2 8 16 32 64 128 256 2>&1 | tail -1
timeout 300 python tools/transpose_probe.py 2>&1 | tail -5
python - <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, torch, paper_2208_06290_b200 as hb
n = 1 << 14
f = hb.factorize(hb.random_hodlr(n, 64, 32, seed=1, s=4.0))
B = np.random.default_rng(0).standard_normal((n, 7))
X = hb.solve(f, B)
Xd = hb.solve(f, torch.from_numpy(B).cuda())
print("numpy multi-RHS == device:", np.array_equal(X, Xd.cpu().numpy()), X.shape, X.flags["C_CONTIGUOUS"])
PY
