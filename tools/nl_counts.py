"""The NL table's preconditioned fixed-point counts (dx = 1e-5,
|u|^2, soliton u0, S0^2): N = 10 / 100 / 500 / 1000 -> printed N_pc
11 / 22 / 25 / 26.  python tools/nl_counts.py [N ...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import swr_inputs as si  # noqa: E402
from paper_1503_02564_b200 import SWR  # noqa: E402

PRINTED = {10: 11, 100: 22, 500: 25, 1000: 26}
for N in [int(a) for a in sys.argv[1:]] or [100, 500, 1000]:
    p = si.config("C4", N=N, dx=1e-5, pinv_exact=1, maxit=2000)
    s = SWR(p, si.inputs(p))
    t0 = time.time()
    s.build()
    st, uT, r = s.solve()
    torch.cuda.synchronize()
    print(f"N={N} dx=1e-5: status {st} N_pc {r['iterations']} (printed {PRINTED.get(N)}) fp_max {r['fp_max']} "
          f"{time.time() - t0:.1f} s", flush=True)
    s.close()
