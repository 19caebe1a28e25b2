"""Table 6 Krylov columns: iterations at which the residual estimate first drops below
rtol * ||b|| for several rtol (from the residual history of one tol = 1e-10 solve)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
rows = [("S0^2", dict(transmission=si.TC_S02)), ("S2^{2,20}", dict(transmission=si.TC_S22, pade_m=20)),
        ("S2^{2,50}", dict(transmission=si.TC_S22, pade_m=50)), ("S2^{2,100}", dict(transmission=si.TC_S22, pade_m=100)),
        ("Robin p=5", dict(transmission=si.TC_ROBIN, robin_p=5.0))]
for name, kw in rows:
    for kname, kry in (("GMRES", si.KRY_GMRES), ("BiCGStab", si.KRY_BICGSTAB)):
        p = si.config("C2", N=2, g0_random=True, krylov=kry, **kw)
        s = SWR(p, si.inputs(p)); s.build(); st, uT, r = s.solve(); torch.cuda.synchronize()
        d, _ = s.get_interface(0)
        bn = float(torch.linalg.norm(d).item())
        h = np.asarray(r["history"], dtype=float) / bn
        out = {}
        for rt in (1e-4, 1e-5, 1e-6, 1e-8, 1e-10):
            idx = np.nonzero(h <= rt)[0] if h.size else []
            out[rt] = int(idx[0]) + 1 if len(idx) else None
        print(f"{name:11s} {kname:8s} total {r['iterations']:4d}  first below rtol: {out}  (||b|| = {bn:.3e})", flush=True)
        del s
