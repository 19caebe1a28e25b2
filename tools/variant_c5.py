"""Time the C5 build + solve with a given libswr variant (tools/build_variant.py)
and compare its u(T) with the product library's.

  python tools/variant_c5.py build_variants/libswr_TAG.so [config]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import swr_inputs as si  # noqa: E402
from paper_1503_02564_b200 import swr  # noqa: E402

name = sys.argv[2] if len(sys.argv) > 2 else "C5"
p = si.config(name)
arrays = si.inputs(p)
res = {}
for tag, L in (("variant", swr.load(os.path.abspath(sys.argv[1]))), ("product", swr.lib())):
    s = swr.SWR(p, arrays, library=L)
    best = None
    for rep in range(4 if tag == "variant" else 1):
        s.build()
        st, uT, r = s.solve()
        torch.cuda.synchronize()
        t = (r["t_build_ms"], r["t_solve_ms"], r["t_march_ms"], r["t_interface_ms"])
        if best is None or sum(t[:2]) < sum(best[:2]):
            best = t
    res[tag] = (uT.copy(), r["iterations"], best)
    s.close()
uv, itv, best = res["variant"]
up, itp, _ = res["product"]
d = float(np.linalg.norm(uv - up) / np.linalg.norm(up))
print(f"{os.path.basename(sys.argv[1])} {name}: it {itv} (product {itp}) build {best[0]:.2f} solve {best[1]:.2f} "
      f"march {best[2]:.2f} toeplitz {best[3]:.2f} ms (best of 4); u(T) vs product {d:.2e}", flush=True)
