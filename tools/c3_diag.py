"""Full-size C3 (and a V(x) twin) sampled sweep errors against the oracle."""
import sys, os
sys.path.insert(0, '.')
import numpy as np, torch, dataclasses
import swr_inputs as si
from paper_1503_02564_b200 import SWR
from oracle import oracle as O
for name, kw in (("C3", {}), ("C3", {"potential": si.POT_VX, "algorithm": si.ALG_NEW})):
    p = dataclasses.replace(si.config(name), **kw)
    arrays = si.inputs(p)
    g_ = SWR(p, arrays)
    Rg, _ = g_.apply_R(None, use_u0=True, want_uT=False)
    Rg = Rg.cpu().numpy()
    o = O.Oracle(p, arrays)
    NT = p.NT
    for j in (27, 28):
        st, ol, orr, _, _ = o.march(j, None, None, use_u0=True)
        a = Rg[(2 * j - 4) * NT:(2 * j - 3) * NT]
        b = Rg[(2 * j - 1) * NT:(2 * j) * NT]
        e1 = np.linalg.norm(a - ol) / np.linalg.norm(ol)
        e2 = np.linalg.norm(b - orr) / max(np.linalg.norm(orr), 1e-300)
        k = np.argmax(np.abs(a - ol))
        print(f"{name} pot={p.potential} march={os.environ.get('SWR_MARCH','res')} j={j} rel_left {e1:.3e} rel_right {e2:.3e} "
              f"worst step {k+1} |ol| {abs(ol[k]):.3e} first-10 err {np.abs(a-ol)[:10].max():.2e}", flush=True)
    del g_
