O=gpurun_out/r02c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "north_star or multi_cta or deterministic" -s -rA > $O/new_tests.txt 2>&1; echo "rc=$?" >> $O/new_tests.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "precond_parity" -s > $O/precond.txt 2>&1
timeout 1200 python tools/c5_gate_experiment.py 1e-10 > $O/c5_gate_mono.txt 2>&1; echo "rc=$?" >> $O/c5_gate_mono.txt
