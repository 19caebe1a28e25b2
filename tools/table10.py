"""The paper's GPU tables (8 K20s, one GPU per subdomain, cuSPARSE):
V = -x^2, S0^2, BiCGStab on the new algorithm's interface problem, zero g0,
dt = 1e-3, N = 2, 4, 8 at dx = 1e-5 and 5e-6 -- here on ONE B200 (build + solve)."""
import sys
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
PAPER = {1e-5: {2: 27.90, 4: 16.13, 8: 12.54}, 5e-6: {2: 51.95, 4: 28.21, 8: 16.30}}
print("# dx N | iterations | build s | solve s | total s | paper (N K20 GPUs) s")
for dx, rows in PAPER.items():
    for N, tp in rows.items():
        p = si.config("C2", N=N, dx=dx, krylov=si.KRY_BICGSTAB)
        s = SWR(p, si.inputs(p))
        for rep in range(2):
            s.build(); st, uT, r = s.solve()
        torch.cuda.synchronize()
        tb, ts = r["t_build_ms"] / 1e3, r["t_solve_ms"] / 1e3
        print(f"{dx:.0e} {N} | {r['iterations']:4d} | {tb:6.2f} | {ts:6.2f} | {tb + ts:6.2f} | {tp}", flush=True)
        del s
