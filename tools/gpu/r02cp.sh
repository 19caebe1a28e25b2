# factor pivot test without hypot: NaN-pivot test, update-inputs test, a parity subset, update timing
O=gpurun_out/r02cp; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "nan_pivot or update_inputs or sweep or vtx or deterministic" -rf > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 300 python tools/e2e_parts.py > $O/parts.txt 2>&1
