O=gpurun_out/r02z; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
SWR_VERBOSE=1 timeout 300 python tools/quick_c5.py C4 > $O/quick_c4.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py tests/test_race_stress.py -q -k "nl or NL or C4 or race or precond" -rf --durations=5 > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
