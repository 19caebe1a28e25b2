# per-CTA phase trace of the C3 marches (constant L0 build, then time-dependent sweeps)
SWR_TRACE_BUILD=1 python paper_1503_02564_b200/_build.py > /dev/null || exit 1
SWR_TRACE_BUILD=1 SWR_TRACE=1 timeout 300 python - <<'PY' 2>&1 | head -60
import sys; sys.path.insert(0, '.')
import torch, swr_inputs as si
from paper_1503_02564_b200 import SWR
p = si.config("C3"); s = SWR(p, si.inputs(p)); s.build(); torch.cuda.synchronize()
PY
python paper_1503_02564_b200/_build.py > /dev/null
