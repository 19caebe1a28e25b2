"""Build-march time of C5 variants (S0^2 vs Robin) to size the history cost."""
import sys, time
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
for tc in (si.TC_S02, si.TC_ROBIN):
    p = si.config("C5", transmission=tc, robin_p=19.0, maxit=1)
    s = SWR(p, si.inputs(p))
    s.build(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t = time.perf_counter(); s.build(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    print("tc", tc, "build ms", [round(x * 1e3, 2) for x in ts])
    del s
