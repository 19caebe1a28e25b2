"""The paper's Tables 4-5 and its nonlinear counterpart: classical
(Algorithm 1 fixed point, N_nopc) vs preconditioned (N_pc: GMRES on
P^{-1}(I - L)g = P^{-1}d for V = 5tx, eqs. 19-20; the preconditioned fixed point
for f(u) = |u|^2, reading A9) iteration counts, S0^2, zero g0, dt = 1e-3, on one
B200.  (The preconditioned fixed point for V = 5tx does not converge within
2000 iterations at N >= 100 on either grid.)"""
import sys
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR

PAPER = {  # (potential, dx): {N: (N_nopc, N_pc)}
    ("V=5tx", 1e-5): {10: (17, 17), 100: (71, 32), 500: (349, 31)},
    ("V=5tx", 1e-4): {10: (17, 17), 100: (71, 32), 500: (349, 26)},
    ("|u|^2", 1e-5): {10: (12, 11), 100: (71, 22), 500: (349, 25)},
    ("|u|^2", 1e-4): {10: (12, 11), 100: (71, 22), 500: (349, 25)},   # the paper's NL table is dx = 1e-5
}
dxs = [float(a) for a in sys.argv[1:]] or [1e-4]
print("# potential dx N | classical FP ours / paper | preconditioned FP ours / paper | device s (cls, pc)")
for (pname, dxp), rows in PAPER.items():
    if dxp not in dxs:
        continue
    pot = si.POT_VTX if pname == "V=5tx" else si.POT_CUBIC
    for N, (pn, pp) in rows.items():
        out = []
        for alg in (si.ALG_CLASSICAL, si.ALG_PRECOND):
            kry = si.KRY_GMRES if (alg == si.ALG_PRECOND and pot == si.POT_VTX) else si.KRY_FIXED_POINT
            if pot == si.POT_CUBIC and 42.0 / (dxp * N) + 1 > 45056:   # no resident NL march beyond 45,056 rows
                out.append(("n/a", 0.0))
                continue
            p = si.config("C3", N=N, dx=dxp, potential=pot, algorithm=alg, krylov=kry, maxit=2000,
                          u0_kind="soliton" if pot == si.POT_CUBIC else "gaussian")
            s = SWR(p, si.inputs(p)); s.build(); st, uT, r = s.solve(); torch.cuda.synchronize()
            out.append((r["iterations"] if st == 0 else f"st{st}", (r["t_build_ms"] + r["t_solve_ms"]) / 1e3))
            del s
        print(f"{pname:6s} {dxp:.0e} {N:4d} | {out[0][0]!s:>5} / {pn:<5} | {out[1][0]!s:>5} / {pp:<5} | "
              f"{out[0][1]:.2f}, {out[1][1]:.2f}", flush=True)
