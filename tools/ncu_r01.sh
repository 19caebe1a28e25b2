# one --set full capture each of the build march, an FFT apply and a CGS pass (k ~ 25), C5
ncu --set full --clock-control none --import-source on -k regex:k_march -c 1 -o gpurun_out/r01_march -f \
    python tools/one_solve.py C5 > gpurun_out/ncu_r01a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fft_conv_reg --launch-skip 25 -c 1 \
    -o gpurun_out/r01_fft -f python tools/one_solve.py C5 > gpurun_out/ncu_r01b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cgs --launch-skip 50 -c 2 \
    -o gpurun_out/r01_cgs -f python tools/one_solve.py C5 > gpurun_out/ncu_r01c.log 2>&1
