O=gpurun_out/r02bg; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/quick_c5.py C4 > /dev/null 2>&1
python - > $O/t.txt 2>&1 <<'PY'
import sys, time; sys.path.insert(0, '.')
import torch, swr_inputs as si
from paper_1503_02564_b200 import SWR
for name in ("C4", "C3"):
    p = si.config(name, pinv_exact=1); s = SWR(p, si.inputs(p))
    for rep in range(2):
        s.build(); st, uT, r = s.solve(); torch.cuda.synchronize()
    print(name, "exact Pinv: status", st, "it", r["iterations"], "build+solve", round(r["t_build_ms"] + r["t_solve_ms"], 1), "ms march", round(r["t_march_ms"], 1))
PY
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py -q -k "pinv or exact or nl or precond" -rf > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
