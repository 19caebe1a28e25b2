# ncu --set full captures of the C5 hot kernels (one launch each) + a launch list of one solve
set -x
python tools/quick_c5.py C5 > gpurun_out/q.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:'k_fft_conv_reg|k_cgs|k_march' -c 5 \
    -o gpurun_out/c5_full -f python tools/quick_c5.py C5 > gpurun_out/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv \
    python tools/one_solve.py C5 > gpurun_out/ncu_list.log 2>&1
