"""Offline check: the oracle's GMRES iteration count at the full C5 size
(single-threaded CPU, ~15-30 min) next to the GPU's."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import swr_inputs as si
from oracle import oracle
p = si.config("C5")
arr = si.inputs(p)
t0 = time.time()
r = oracle.Oracle(p, arr).solve()
t1 = time.time()
print(f"oracle C5: status {r['status']} iterations {r['iterations']} time {t1 - t0:.0f} s", flush=True)
np.save("/tmp/oracle_c5_uT.npy", r["uT"])   # 67 MB: kept off gpurun_out (64 MiB limit)
np.save("gpurun_out/oracle_c5_hist.npy", np.array(r["history"]))
try:
    import torch
    from paper_1503_02564_b200 import SWR
    s = SWR(p, arr)
    st, uT, rg = s.solve()
    err = np.linalg.norm(uT - r["uT"]) / np.linalg.norm(r["uT"])
    h = np.array(rg["history"])
    print(f"gpu C5: status {st} iterations {rg['iterations']} rel L2 vs oracle {err:.3e}", flush=True)
    np.save("gpurun_out/gpu_c5_hist.npy", h)
except Exception as e:
    print("gpu part failed:", e)
