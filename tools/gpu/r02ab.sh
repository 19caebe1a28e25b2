O=gpurun_out/r02ab; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "c5_full" -s -rf > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
