"""One C5 build + solve (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
p = si.config(sys.argv[1] if len(sys.argv) > 1 else "C5")
s = SWR(p, si.inputs(p))
s.build()
st, uT, r = s.solve()
torch.cuda.synchronize()
print("iters", r["iterations"])
