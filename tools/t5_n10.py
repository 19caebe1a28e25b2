"""The paper's T5 row N = 10 at dx = 1e-5 (|u|^2, soliton u0, preconditioned
fixed point, S0^2): N_j = 420,001, the streaming NL march.
Prints the outer count (the paper prints N_pc = 11) and the timings.
Also times one R_nl sweep.  python tools/t5_n10.py [pinv_exact]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import swr_inputs as si  # noqa: E402
from paper_1503_02564_b200 import SWR  # noqa: E402

pe = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = si.Problem(dx=1e-5, dt=1e-3, N=10, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND, krylov=si.KRY_FIXED_POINT,
               u0_kind="soliton", pinv_exact=pe)
s = SWR(p, si.inputs(p))
t0 = time.time()
Rg, _ = s.apply_R(torch.zeros(p.ng, dtype=torch.complex128, device="cuda"), use_u0=True)
torch.cuda.synchronize()
print(f"one R_nl sweep: {time.time() - t0:.2f} s", flush=True)
t0 = time.time()
s.build()
st, uT, r = s.solve()
torch.cuda.synchronize()
print(f"T5 N=10 dx=1e-5 (pinv_exact={pe}): status {st} outer {r['iterations']} (paper N_pc 11) inner {r['inner_iterations']} "
      f"fp_max {r['fp_max']} wall {time.time() - t0:.1f} s march {r['t_march_ms'] / 1e3:.1f} s", flush=True)
