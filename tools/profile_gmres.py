"""C5 build + a short GMRES (maxit from argv) for ncu launch lists / captures."""
import sys
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 40
p = si.config("C5", maxit=maxit)
s = SWR(p, si.inputs(p))
s.build()
st, uT, r = s.solve()
torch.cuda.synchronize()
print("iters", r["iterations"], "solve ms", r["t_solve_ms"], "intf ms", r["t_interface_ms"], "march ms", r["t_march_ms"])
