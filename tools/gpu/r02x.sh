# four-warp FFT apply + streaming NL march
O=gpurun_out/r02x; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for cfg in C5 N100; do
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_fft_conv_reg --csv --log-file $O/fft_${cfg}.csv python tools/fft_probe.py $cfg 40 > $O/log_${cfg}.txt 2>&1
done
timeout 300 python tools/quick_c5.py C5 > $O/quick_c5.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py tests/test_race_stress.py -q -x -k "interface_operator or new_algorithm or toeplitz or multirank or logical or precond or pinv or stream or nl or race or c5_full or deterministic or solver" -rf --durations=5 > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
