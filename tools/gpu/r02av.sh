O=gpurun_out/r02av; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py tests/test_race_stress.py -q -k "stream or nl or race or edge or N10" -rf --durations=5 > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 900 python tools/t5_n10.py 1 > $O/t5.txt 2>&1
