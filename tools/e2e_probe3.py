"""Where does the slow e2e iteration lose time (dev probe): copy-stream finish vs compute finish."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
from paper_2208_06290_b200 import hodlr as hm
n, m, r = 1 << 20, 64, 32
h0 = hb.random_hodlr(n, m, r, seed=0, s=1.0)
Dh, Uh, Vh = h0.D.cpu().pin_memory(), h0.U.cpu().pin_memory(), h0.V.cpu().pin_memory()
del h0
torch.cuda.empty_cache()
st = torch.cuda.current_stream()
for it in range(9):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e0.record(st)
    t0 = time.perf_counter()
    f = hb.factorize_from_host(n, m, r, Dh, Uh, Vh, check=False)
    t_enq = time.perf_counter()
    cs = hm._COPY_STREAMS[str(torch.device("cuda"))]
    ec = torch.cuda.Event(enable_timing=True); ec.record(cs)
    ef = torch.cuda.Event(enable_timing=True); ef.record(st)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"it {it}: wall {1e3 * (t1 - t0):.1f} ms  enqueue {1e3 * (t_enq - t0):.1f} ms  copies done at {e0.elapsed_time(ec):.1f} ms"
          f"  compute done at {e0.elapsed_time(ef):.1f} ms", flush=True)
    del f
