"""One build + solve of a config (for ncu launch lists).
  python tools/one_solve.py [config] [field=value ...]   e.g. C4 pinv_exact=1"""
import sys
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
kw = {}
for a in sys.argv[2:]:
    k, v = a.split("=", 1)
    kw[k] = int(v) if v.lstrip("-").isdigit() else float(v)
p = si.config(sys.argv[1] if len(sys.argv) > 1 else "C5", **kw)
s = SWR(p, si.inputs(p))
s.build()
st, uT, r = s.solve()
torch.cuda.synchronize()
print("iters", r["iterations"])
