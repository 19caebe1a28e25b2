O=gpurun_out/r02g; mkdir -p $O
for v in d e f; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so >> $O/variants.txt 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r1_launches.csv bash -c "cd build_variants/r1_tree && python tools/one_solve.py C5" > $O/ncu_r1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cur_launches.csv python tools/one_solve.py C5 > $O/ncu_cur.log 2>&1
gzip -f $O/*.csv
timeout 900 python -m pytest tests/test_multirank.py tests/test_gpu_parity.py -q -x -k "stream or cgs or logical or deterministic or new_algorithm or precond or solver" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
