# streaming march: thread-interleaved scratch layout
O=gpurun_out/r02au; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/quick_c5.py C2 > $O/quick_c2.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py tests/test_race_stress.py -q -k "stream or c2 or higher_order or race or logical or edge" -rf --durations=5 > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
