# TDM march: one rhs pass per step + carry fix-up
O=gpurun_out/r02t; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/quick_c5.py C3 > $O/quick_c3.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py tests/test_race_stress.py -q -k "vtx or precond or C3 or paper_iteration or race or solver" -rf > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
