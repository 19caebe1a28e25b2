"""The stagnating restarted-GMRES case of tools/robustness_check.py (Robin
p = 19, N_T = 700, ~60 restart cycles): iteration counts and u(T) of the two
oracle builds (default and FMA contraction) -- the rounding spread the GPU's
count is compared with.  python tools/robustness_fma.py"""
import sys

import numpy as np

sys.path.insert(0, '.')
import swr_inputs as si  # noqa: E402
from oracle import oracle  # noqa: E402

p = si.Problem(a0=-6, b0=6, T=0.35, dx=0.02, dt=5e-4, N=5, potential=si.POT_VX, transmission=si.TC_ROBIN,
               robin_p=19.0)
arr = si.inputs(p)
x = p.nodes()
arr["u0"] = np.exp(-(x + 1) ** 2 + 3j * x)
oracle.set_threads(8)
a = oracle.Oracle(p, arr).solve()
b = oracle.Oracle(p, arr, library=oracle.lib_fma()).solve()
rel = np.linalg.norm(a["uT"] - b["uT"]) / np.linalg.norm(a["uT"])
print(f"oracle default {a['iterations']} iterations, FMA build {b['iterations']}, u(T) apart {rel:.2e}")
