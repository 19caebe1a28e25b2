# stored b_k in the two-pass streaming march only: C2, NL sweep, streaming tests
O=gpurun_out/r02cf; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/quick_c5.py C2 > $O/quick_c2.txt 2>&1
timeout 300 python tools/nl_stream_time.py > $O/nls.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py tests/test_race_stress.py -q -k "stream or c2 or nl or race or edge or logical" -rf --durations=5 > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
