O=gpurun_out/r02j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/quick_c5.py C5 > $O/quick_c5.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rf --durations=10 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
