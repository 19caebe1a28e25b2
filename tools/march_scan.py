"""Time the build march for several subdomain counts (launch shapes)."""
import sys, time
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
for N in [int(a) for a in sys.argv[1:]] or [500, 1000, 2000]:
    p = si.config("C5", N=N, maxit=1)
    s = SWR(p, si.inputs(p))
    s.build(); torch.cuda.synchronize()
    t = time.perf_counter(); s.build(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    cells = (3 * N - 2) * p.Nj * p.NT
    print(f"N={N} Nj={p.Nj} build {dt*1e3:.2f} ms  {cells/dt/1e9:.1f} Gcell-steps/s")
    del s
