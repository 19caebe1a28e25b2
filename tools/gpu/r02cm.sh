# update-inputs test incl. device buffers
O=gpurun_out/r02cm; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "update_inputs" -rf > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
