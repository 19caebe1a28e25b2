"""One R_nl sweep at the paper's T5 N = 10 size (N_j = 420,001, the streaming
NL march) with a given libswr build.  python tools/nl_stream_time.py [lib]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import swr_inputs as si  # noqa: E402
from paper_1503_02564_b200 import swr  # noqa: E402

L = swr.load(os.path.abspath(sys.argv[1])) if len(sys.argv) > 1 else None
p = si.Problem(dx=1e-5, dt=1e-3, N=10, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND, u0_kind="soliton")
s = swr.SWR(p, si.inputs(p), library=L)
z = torch.zeros(p.ng, dtype=torch.complex128, device="cuda")
s.apply_R(z, use_u0=True)
best = 1e9
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.time()
    s.apply_R(z, use_u0=True)
    torch.cuda.synchronize()
    best = min(best, time.time() - t0)
print(f"{os.path.basename(sys.argv[1]) if len(sys.argv) > 1 else 'product'}: one R_nl sweep {best * 1e3:.1f} ms")
