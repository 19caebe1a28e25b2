"""Time the register-FFT Toeplitz apply (I - L)x alone: NEW build of a config,
then `reps` applies (run under ncu --cache-control none for warm per-launch
durations).  python tools/fft_probe.py [config] [reps] [--lib=path]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import swr_inputs as si  # noqa: E402
from paper_1503_02564_b200 import swr  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "C5"
reps = int(args[1]) if len(args) > 1 else 50
libp = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--lib=")), None)
p = si.config(name) if name != "N100" else si.config("C5", N=100)
s = swr.SWR(p, si.inputs(p), library=swr.load(os.path.abspath(libp)) if libp else None)
s.build()
x = torch.randn(s.ng, dtype=torch.complex128, device="cuda")
for _ in range(reps):
    y = s.apply_I_minus_L(x, 0)
torch.cuda.synchronize()
print("ok", float(y.abs().sum()))
