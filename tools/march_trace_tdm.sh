# TDM march copy latency (trace slot 28: prefetch issue -> data ready, cycles) at
# two cluster sizes: C3 (N = 100, N_j = 42,001, CS = 15) and N = 1000 (N_j = 4201)
SWR_TRACE_BUILD=1 python paper_1503_02564_b200/_build.py > /dev/null || exit 1
for N in 100 1000; do
SWR_TRACE_BUILD=1 SWR_TRACE=1 N=$N timeout 300 python - <<'PY' 2>&1 | grep -A3 "march trace" | tail -4
import os, sys; sys.path.insert(0, '.')
import torch, swr_inputs as si
from paper_1503_02564_b200 import SWR
p = si.config("C3", N=int(os.environ["N"])); s = SWR(p, si.inputs(p)); s.build(); torch.cuda.synchronize()
PY
done
python paper_1503_02564_b200/_build.py > /dev/null
