O=gpurun_out/r02u; mkdir -p $O
bash tools/march_trace_tdm.sh > $O/trace_tdm.txt 2>&1
SWR_TRACE_BUILD=1 python paper_1503_02564_b200/_build.py > /dev/null
SWR_TRACE_BUILD=1 SWR_TRACE=1 timeout 300 python - > $O/trace_tdm_full.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import torch, swr_inputs as si
from paper_1503_02564_b200 import SWR
p = si.config("C3"); s = SWR(p, si.inputs(p)); s.build(); torch.cuda.synchronize()
PY
python paper_1503_02564_b200/_build.py > /dev/null
