O=gpurun_out/r02r; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for cfg in C5 N100; do
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_fft_conv_reg --csv --log-file $O/fft_${cfg}.csv python tools/fft_probe.py $cfg 40 > $O/log_${cfg}.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py -q -x -k "interface_operator or new_algorithm or toeplitz or multirank or logical or precond or pinv" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 300 python tools/quick_c5.py C5 > $O/quick_c5.txt 2>&1
