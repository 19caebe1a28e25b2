O=gpurun_out/r02d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests/test_multirank.py -q -x -k "new-gmres" > $O/mr_quick.txt 2>&1; echo "rc=$?" >> $O/mr_quick.txt
timeout 1500 python -m pytest tests -q -m gpu -rf --durations=15 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 300 python tools/quick_c5.py C5 > $O/quick_c5.txt 2>&1
