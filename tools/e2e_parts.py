"""Where the C5 e2e overhead goes: stream-timed swr_update_inputs (host u0 +
V_x, each alone), the raw pinned copies, and a solve into host vs device
memory.  python tools/e2e_parts.py [lib]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import swr_inputs as si  # noqa: E402
from paper_1503_02564_b200 import SWR, swr  # noqa: E402

lib = swr.load(sys.argv[1]) if len(sys.argv) > 1 else None
p = si.config("C5")
arr = si.inputs(p)
st = torch.cuda.Stream()
s = SWR(p, arr, stream=st, library=lib)
u0 = torch.from_numpy(arr["u0"]).pin_memory()
vx = torch.from_numpy(arr["V_x"]).pin_memory()
outh = torch.empty(p.Nx + 1, dtype=torch.complex128).pin_memory()
outd = torch.empty(p.Nx + 1, dtype=torch.complex128, device="cuda")
du0 = torch.empty_like(u0, device="cuda")
dvx = torch.empty_like(vx, device="cuda")


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            fn()
            b.record(st)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


with torch.cuda.stream(st):
    s.build()
    s.solve(out=outd)
print(f"raw H2D u0 67 MB      {timed(lambda: du0.copy_(u0, non_blocking=True)):.3f} ms")
print(f"raw H2D V_x 34 MB     {timed(lambda: dvx.copy_(vx, non_blocking=True)):.3f} ms")
print(f"raw D2H u(T) 67 MB    {timed(lambda: outh.copy_(outd, non_blocking=True)):.3f} ms")
print(f"update u0 + V_x       {timed(lambda: s.update_inputs(u0=u0, V_x=vx)):.3f} ms")
print(f"update u0 only        {timed(lambda: s.update_inputs(u0=u0)):.3f} ms")
print(f"update V_x only       {timed(lambda: s.update_inputs(V_x=vx)):.3f} ms")


def solve_to(out):
    s.build()
    s.solve(out=out.numpy() if out.device.type == "cpu" else out)


print(f"build + solve, device out {timed(lambda: solve_to(outd)):.3f} ms")
print(f"build + solve, host out   {timed(lambda: solve_to(outh)):.3f} ms")
