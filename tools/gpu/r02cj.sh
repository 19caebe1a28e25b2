# u0 copy overlapping the factorisation in swr_update_inputs: update-inputs test, e2e
O=gpurun_out/r02cj; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "update_inputs or deterministic" -rf > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extra > $O/bench$i.json 2> $O/bench$i.err; done
