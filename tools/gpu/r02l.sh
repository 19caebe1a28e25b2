# K = 3 build march + 256-thread fixed-order reduce: C5 timing vs march_form 2, parity subsets, launch list
O=gpurun_out/r02l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python tools/k3_check.py C5 --oracle > $O/k3_c5.txt 2>&1; echo "rc=$?" >> $O/k3_c5.txt
timeout 300 python tools/quick_c5.py C5 > $O/quick_c5.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py -q -x -k "interface_operator or new_algorithm or c5_full or multirank or logical or deterministic or solver_variant or edge or sweep_R" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/one_solve.py C5 > $O/ncu_list.log 2>&1
gzip -f $O/launches.csv
R=/tmp/rep; mkdir -p $R
ncu --set full --clock-control none --import-source on -k regex:'k_march' -c 1 -o $R/march3 -f python tools/one_solve.py C5 > $O/ncu_m.log 2>&1
python tools/ncu_brief.py $R/march3.ncu-rep > $O/ncu_march3.txt 2>&1
cp $R/march3.ncu-rep $O/ 2>/dev/null
