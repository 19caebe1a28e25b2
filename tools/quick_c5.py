import time, sys, numpy as np, torch
sys.path.insert(0, '.')
import swr_inputs as si
from paper_1503_02564_b200 import SWR, swr
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
lib = swr.load(sys.argv[2]) if len(sys.argv) > 2 else None   # optional variant library
p = si.config(name)
arr = si.inputs(p)
t0 = time.time(); s = SWR(p, arr, library=lib); torch.cuda.synchronize(); print("setup", time.time() - t0)
for rep in range(2):
    t0 = time.time(); s.build(); st, uT, r = s.solve(); t1 = time.time() - t0
    print(f"status {st} iters {r['iterations']} wall {t1:.3f}s build {r['t_build_ms']:.2f}ms solve {r['t_solve_ms']:.2f}ms march {r['t_march_ms']:.2f}ms intf {r['t_interface_ms']:.2f}ms cell_steps {r['cell_steps']:.3e} marches {r['n_marches']} launches {r['n_kernel_launches']}")
    print("  march Gcell-steps/s", r['cell_steps'] / r['t_march_ms'] / 1e6, " HBM-equiv frac", 32 * r['cell_steps'] / (r['t_march_ms'] * 1e-3) / 6538.6e9)
