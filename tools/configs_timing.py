"""One build + solve of each BASELINE config (C2..C5) on the GPU: times, iterations."""
import sys, time
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
for name in (sys.argv[1:] or ["C2", "C3", "C4", "C5"]):
    p = si.config(name)
    t0 = time.perf_counter()
    s = SWR(p, si.inputs(p))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s.build()
    st, uT, r = s.solve()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: N={p.N} Nj={p.Nj} NT={p.NT} setup {t1-t0:.2f}s build {r['t_build_ms']:.1f}ms "
          f"solve {r['t_solve_ms']:.1f}ms (wall {t2-t1:.2f}s) status {st} outer {r['iterations']} "
          f"inner {r['inner_iterations']} fp_max {r['fp_max']} march {r['t_march_ms']:.1f}ms "
          f"intf {r['t_interface_ms']:.1f}ms marches {r['n_marches']} Gcs/s {r['cell_steps']/max(r['t_march_ms'],1e-9)/1e6:.1f}",
          flush=True)
    del s
