# final head sanity: smoke, C5 quick, determinism and update tests
O=gpurun_out/r02cv; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 300 python tools/quick_c5.py C5 > $O/c5.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "deterministic or update_inputs or nan_pivot or c5_north" -rf > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
