# two-pass streaming NL march; the paper's T5 N = 10 row at dx = 1e-5
O=gpurun_out/r02al; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py tests/test_race_stress.py -q -k "stream or nl or race" -rf --durations=5 > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
SWR_VERBOSE=1 timeout 1500 python tools/t5_n10.py 1 > $O/t5.txt 2>&1; echo "rc=$?" >> $O/t5.txt
