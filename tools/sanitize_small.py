"""Small-shape runs of the cluster / DSMEM / st.async / mbarrier kernels for
compute-sanitizer (racecheck, synccheck, memcheck): the resident march with a
3-CTA cluster (N_j = 8401, the C5 subdomain size, 11 rows per thread), the
nonlinear march (multi-CTA cluster) and the streaming march (a 3-CTA chain),
each a handful of time steps so the instrumented run stays short.

  compute-sanitizer --tool racecheck python tools/sanitize_small.py [which]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import swr_inputs as si  # noqa: E402
from paper_1503_02564_b200 import SWR  # noqa: E402


def gauss(p):
    x = p.nodes()
    return np.exp(-(x * x) / 1e-3 + 2j * x)


def run(name, p, env=None):
    for k in ("SWR_MARCH",):
        os.environ.pop(k, None)
    for k, v in (env or {}).items():
        os.environ[k] = v
    arrays = si.inputs(p)
    arrays["u0"] = gauss(p)
    s = SWR(p, arrays)
    rng = np.random.default_rng(1)
    g = torch.as_tensor(rng.standard_normal(p.ng) + 1j * rng.standard_normal(p.ng), device="cuda")
    Rg, uT = s.apply_R(g, use_u0=True, want_uT=True)
    torch.cuda.synchronize()
    print(name, "ok", float(Rg.abs().max()), float(uT.abs().max()), flush=True)
    s.close()


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    # resident march, C5 subdomain size N_j = 8401 -> M = 11, P = 256, CS = 3
    if which in ("all", "march"):
        run("k_march CS=3", si.Problem(a0=-0.42, b0=0.42, T=4e-3, dx=1e-5, dt=1e-3, N=10, potential=si.POT_VX))
    # time-dependent factors (the TDM variant with per-step bulk copies)
    if which in ("all", "tdm"):
        run("k_march TDM", si.Problem(a0=-0.42, b0=0.42, T=4e-3, dx=1e-5, dt=1e-3, N=10, potential=si.POT_VTX,
                                      algorithm=si.ALG_PRECOND))
    # nonlinear march (multi-CTA cluster, cluster-wide fixed-point stop)
    if which in ("all", "nl"):
        run("k_march_nl", si.Problem(a0=-0.42, b0=0.42, T=3e-3, dx=1e-5, dt=1e-3, N=10, potential=si.POT_CUBIC,
                                     algorithm=si.ALG_PRECOND))
    # streaming march (chain of co-resident CTAs, global-memory flags)
    if which in ("all", "stream"):
        run("k_march_stream", si.Problem(a0=-0.42, b0=0.42, T=4e-3, dx=1e-5, dt=1e-3, N=10, potential=si.POT_VX),
            env={"SWR_MARCH": "stream"})


if __name__ == "__main__":
    main()
