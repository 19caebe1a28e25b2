"""C3 / C4 with the inner-Krylov P^{-1} (paper) vs the exact causal P^{-1} (8(f)-4)."""
import sys, dataclasses
sys.path.insert(0, '.')
import numpy as np, torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
for name in (sys.argv[1:] or ["C3", "C4"]):
    out = {}
    for ex in (0, 1):
        p = dataclasses.replace(si.config(name), pinv_exact=ex)
        s = SWR(p, si.inputs(p))
        for rep in range(2):
            s.build()
            st, uT, r = s.solve()
        torch.cuda.synchronize()
        out[ex] = uT
        print(f"{name} pinv_exact={ex}: status {st} outer {r['iterations']} inner {r['inner_iterations']} "
              f"build {r['t_build_ms']:.1f} ms solve {r['t_solve_ms']:.1f} ms march {r['t_march_ms']:.1f} ms "
              f"intf {r['t_interface_ms']:.1f} ms launches {r['n_kernel_launches']}", flush=True)
        del s
    print(f"{name}: ||u_exact - u_krylov|| / ||u|| = {np.linalg.norm(out[1] - out[0]) / np.linalg.norm(out[0]):.2e}")
