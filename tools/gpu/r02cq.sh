# final head: smoke, bench, launch list, full GPU suite
O=gpurun_out/r02cq; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extra > $O/ncu_list.log 2>&1
gzip -f $O/launches.csv
timeout 2400 python -m pytest tests -q -m gpu -rf --durations=10 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
