# norm reduce fused into the next Toeplitz apply
O=gpurun_out/r02ak; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/quick_c5.py C5 > $O/quick_c5.txt 2>&1
timeout 300 python tools/quick_c5.py C4 > $O/quick_c4.txt 2>&1
timeout 300 python tools/quick_c5.py C3 > $O/quick_c3.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rf --durations=5 > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
