# round-2 profile set: bench line, bench launch list, ncu --set full of the top kernels (text summaries only)
O=gpurun_out/r02ah; mkdir -p $O
R=/tmp/rep; mkdir -p $R
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extra > $O/ncu_list.log 2>&1
gzip -f $O/launches.csv
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:'k_march<' -c 1 -o $R/march -f python tools/one_solve.py C5 > $O/n1.log 2>&1
$NCU -k regex:k_fft_conv_reg --launch-skip 400 -c 1 -o $R/fft -f python tools/one_solve.py C5 > $O/n2.log 2>&1
$NCU -k regex:'k_cgs<8' --launch-skip 200 -c 1 -o $R/cgs -f python tools/one_solve.py C5 > $O/n3.log 2>&1
$NCU -k regex:k_cgs_axpy --launch-skip 400 -c 1 -o $R/axpy -f python tools/one_solve.py C5 > $O/n4.log 2>&1
$NCU -k regex:k_cgs_reduce --launch-skip 800 -c 1 -o $R/reduce -f python tools/one_solve.py C5 > $O/n5.log 2>&1
$NCU -k regex:k_march_nl -c 1 -o $R/nl -f python tools/one_solve.py C4 > $O/n6.log 2>&1
$NCU -k regex:'k_march<11, 1, 256, 1' -c 1 -o $R/tdm -f python tools/one_solve.py C3 > $O/n7.log 2>&1
$NCU -k regex:k_march_stream2 -c 1 -o $R/stream2 -f python tools/one_solve.py C2 > $O/n8.log 2>&1
for r in march fft cgs axpy reduce nl tdm stream2; do echo "######## $r" >> $O/ncu_brief.txt; python tools/ncu_brief.py $R/$r.ncu-rep >> $O/ncu_brief.txt 2>&1; python tools/ncu_summary.py $R/$r.ncu-rep >> $O/ncu_full_$r.txt 2>&1; done
for r in march fft; do ncu -i $R/$r.ncu-rep --page raw --csv > $O/raw_$r.csv 2>/dev/null; done
gzip -f $O/raw_*.csv
ls -la $O
