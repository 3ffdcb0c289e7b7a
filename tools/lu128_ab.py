"""Bitwise A/B of the s = 128 K-block LU variants (dev check): run twice with
HODLR_LU128 unset / =sr, compare K, Kinv, pivots, Y; then time the cfg3-shape factor."""
import os, subprocess, sys, time
sys.path.insert(0, ".")
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import numpy as np, torch
    import paper_2208_06290_b200 as hb
    n, m, r = 1 << 16, 64, 64
    h = hb.random_hodlr(n, m, r, seed=3, s=16.0)
    f = hb.factorize(h, check=False)
    np.savez(sys.argv[2], K=f.K.cpu().numpy(), Kinv=f.Kinv.cpu().numpy(), ks=f.kswaps.cpu().numpy(),
             kp=f.kperm.cpu().numpy(), ki=f.kinfo.cpu().numpy(), Y=f.Y.cpu().numpy())
    n = 1 << 21
    h0 = hb.random_hodlr(n, m, r, seed=0, s=1.0)
    ts = []
    for it in range(3):
        hh = h0.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
        hb.factorize(hh, check=False); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        del hh
    print(os.environ.get("HODLR_LU128", "reg"), "cfg3-shape factor ms", [round(1e3 * x, 1) for x in ts], flush=True)
    sys.exit(0)
import numpy as np
env = dict(os.environ); env.pop("HODLR_LU128", None)
subprocess.run([sys.executable, __file__, "run", "/tmp/lu_reg.npz"], env=env, check=True)
subprocess.run([sys.executable, __file__, "run", "/tmp/lu_sr.npz"], env=dict(env, HODLR_LU128="sr"), check=True)
a, b = np.load("/tmp/lu_reg.npz"), np.load("/tmp/lu_sr.npz")
for k in a.files:
    print(k, "bitwise equal" if a[k].tobytes() == b[k].tobytes() else f"DIFFER (max {np.abs(a[k] - b[k]).max()})")
