"""North-star gate experiment at C5 (N = 500, dx = 1e-5, N_T = 500): the GPU
solve against the threaded oracle (and the oracle built with FMA, whose only
difference is rounding) at the paper's tolerance and tighter ones.

  python tools/c5_gate_experiment.py [tol ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import swr_inputs as si  # noqa: E402
from oracle import oracle  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    import torch
    from paper_1503_02564_b200 import SWR
    tols = [float(t) for t in sys.argv[1:]] or [1e-10, 1e-12]
    P = os.cpu_count()
    for tol in tols:
        p = si.config("C5", tol=tol, maxit=3000)
        arrays = si.inputs(p)
        s = SWR(p, arrays)
        s.build()
        st, uT, rg = s.solve()
        g_gpu = s.get_g().cpu().numpy()
        s.close()
        torch.cuda.synchronize()
        out = {}
        for name, lib in (("oracle", oracle.lib()), ("oracle_fma", oracle.lib_fma())):
            if name == "oracle_fma" and tol != tols[0]:
                continue
            oracle.set_threads(P, lib)
            t0 = time.time()
            ro = oracle.Oracle(p, arrays, library=lib).solve()
            out[name] = (ro, time.time() - t0)
        ro, t_o = out["oracle"]
        h_g, h_o = rg["history"], ro["history"]
        n = min(len(h_g), len(h_o))
        r0 = float(np.linalg.norm(si.inputs(p)["u0"]))  # scale only for printing
        print(f"tol {tol:g}: GPU status {st} it {rg['iterations']} | oracle status {ro['status']} it "
              f"{ro['iterations']} ({t_o:.1f} s on {P} threads)")
        print(f"  residual estimates: max |gpu - oracle| / h_0 = {np.abs(h_g[:n] - h_o[:n]).max() / h_o[0]:.3e}, "
              f"final gpu {h_g[-1] / h_o[0]:.3e} oracle {h_o[-1] / h_o[0]:.3e} (relative to h_0)")
        print(f"  u(T): rel(gpu, oracle) = {rel(uT, ro['uT']):.3e}; g: {rel(g_gpu, ro['g']):.3e}")
        if tol == tols[0]:
            # the monodomain solve on the same grid (N = 1: one march, no interface
            # problem): the exact discrete solution the SWR iteration converges to
            q = si.config("C5", N=1)
            oracle.set_threads(1)
            t0 = time.time()
            st_m, um, _ = oracle.Oracle(q, arrays).monodomain()
            out["mono"] = um
            print(f"  monodomain (oracle, {time.time() - t0:.1f} s): rel(gpu, mono) = {rel(uT, um):.3e}, "
                  f"rel(oracle, mono) = {rel(ro['uT'], um):.3e}, "
                  f"rel(oracle_fma, mono) = {rel(out['oracle_fma'][0]['uT'], um):.3e}")
        if "oracle_fma" in out:
            rf, t_f = out["oracle_fma"]
            print(f"  oracle_fma: it {rf['iterations']}; u(T) rel(fma, oracle) = {rel(rf['uT'], ro['uT']):.3e}, "
                  f"rel(gpu, fma) = {rel(uT, rf['uT']):.3e}; g rel(fma, oracle) = {rel(rf['g'], ro['g']):.3e}")
        sys.stdout.flush()


if __name__ == "__main__":
    main()
