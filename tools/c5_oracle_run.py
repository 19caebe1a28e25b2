"""Run the threaded CPU oracle on C5 (or another config) and save u(T), g,
the residual history and the counts (npz): the reference side of the
north-star gate experiments.

  python tools/c5_oracle_run.py OUT.npz [--config C5] [--tol 1e-10] [--fma] [--threads P]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import swr_inputs as si  # noqa: E402
from oracle import oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--config", default="C5")
ap.add_argument("--tol", type=float, default=1e-10)
ap.add_argument("--maxit", type=int, default=2000)
ap.add_argument("--fma", action="store_true")
ap.add_argument("--threads", type=int, default=os.cpu_count())
a = ap.parse_args()
p = si.config(a.config, tol=a.tol, maxit=a.maxit)
lib = oracle.lib_fma() if a.fma else oracle.lib()
oracle.set_threads(a.threads, lib)
t0 = time.time()
r = oracle.Oracle(p, si.inputs(p), library=lib).solve()
dt = time.time() - t0
np.savez(a.out, uT=r["uT"], g=r["g"], history=r["history"], iterations=r["iterations"], status=r["status"],
         seconds=dt, threads=a.threads, tol=a.tol)
print(f"{a.config} tol={a.tol:g} fma={a.fma} threads={a.threads}: status {r['status']} it {r['iterations']} "
      f"{dt:.1f} s", flush=True)
