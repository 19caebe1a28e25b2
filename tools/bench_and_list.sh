# bench line (default config) + ncu launch list of one C5 build+solve
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv \
    python tools/one_solve.py C5 > gpurun_out/ncu_list.log 2>&1
