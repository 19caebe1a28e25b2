# Round profile refresh (one GPU): bench lines, the ncu launch list of the
# bench command, and --set full captures of the top kernels (summaries only
# come back: the .ncu-rep files stay in /tmp on the box).
O=gpurun_out/prof; mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py $O/bench_launches.csv > $O/bench_launches.txt
gzip -f $O/bench_launches.csv
R=/tmp/rep; mkdir -p $R
ncu --set full --clock-control none --import-source on -k regex:k_march -c 1 -o $R/march -f \
    python tools/one_solve.py C5 > $O/ncu_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fft_conv_reg --launch-skip 25 -c 1 -o $R/fft -f \
    python tools/one_solve.py C5 > $O/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_cgs<' --launch-skip 50 -c 1 -o $R/cgs_dots -f \
    python tools/one_solve.py C5 > $O/ncu_c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cgs_axpy --launch-skip 50 -c 1 -o $R/cgs_axpy -f \
    python tools/one_solve.py C5 > $O/ncu_d.log 2>&1
python tools/ncu_brief.py $R/march.ncu-rep $R/fft.ncu-rep $R/cgs_dots.ncu-rep $R/cgs_axpy.ncu-rep > $O/ncu_summary.txt 2>&1
ls -la $O
