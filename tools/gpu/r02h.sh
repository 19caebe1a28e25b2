O=gpurun_out/r02h; mkdir -p $O
for v in d2 g j k; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so >> $O/variants.txt 2>&1; done
timeout 600 python -m pytest tests/test_race_stress.py -q > $O/race.txt 2>&1; echo "rc=$?" >> $O/race.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
