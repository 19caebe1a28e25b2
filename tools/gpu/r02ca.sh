# bench other_configs with the C5 handle freed first
O=gpurun_out/r02ca; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
