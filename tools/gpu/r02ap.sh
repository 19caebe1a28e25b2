O=gpurun_out/r02ap; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/quick_c5.py C5 > $O/quick_c5.txt 2>&1
bash tools/march_trace.sh > $O/trace_c5.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py tests/test_race_stress.py -q -k "sweep_R or interface_operator or new_algorithm or higher_order or race or deterministic or logical or c5_full or edge or solver" -rf --durations=5 > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
