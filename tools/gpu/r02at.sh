O=gpurun_out/r02at; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "edge" -rf > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
