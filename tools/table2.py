"""The paper's Tables 2-3 experiment (V = -x^2, dt = 1e-3, dx = 1e-5,
S0^2, zero g0, N = 2 .. 500): the classical and the new algorithm with the fixed
point, GMRES and BiCGStab, on one B200.  Iterations and device times (ms)
beside the paper's times (seconds on N cores: T_cls / T_new)."""
import sys
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR

PAPER_FP = {2: (773.07, 773.72), 10: (2937.77, 178.30), 100: (359.30, 18.19), 500: (284.78, 4.76)}
print("# N | algorithm + solver | iterations | build ms | solve ms | paper (FP: T_cls / T_new s)")
for N in (2, 10, 100, 500):
    for alg, aname in ((si.ALG_NEW, "new"), (si.ALG_CLASSICAL, "classical")):
        for kry, kname in ((si.KRY_FIXED_POINT, "FP"), (si.KRY_GMRES, "GMRES"), (si.KRY_BICGSTAB, "BiCGStab")):
            p = si.config("C5", N=N, algorithm=alg, krylov=kry, maxit=2000)
            s = SWR(p, si.inputs(p))
            s.build()
            st, uT, r = s.solve()
            torch.cuda.synchronize()
            it = r["iterations"] if st == 0 else f"st{st}"
            print(f"{N:4d} | {aname:9s} {kname:8s} | {it!s:>5} | {r['t_build_ms']:8.1f} | {r['t_solve_ms']:9.1f} | "
                  f"{PAPER_FP[N] if kry == si.KRY_FIXED_POINT else ''}", flush=True)
            del s
