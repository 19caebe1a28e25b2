O=gpurun_out/r02p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for cfg in C5 N100; do
for v in product nofc nox nofcx; do
  L=""; [ $v != product ] && L="--lib=build_variants/libswr_$v.so"
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_fft_conv_reg --csv --log-file $O/fft_${cfg}_$v.csv python tools/fft_probe.py $cfg 40 $L > $O/log_${cfg}_$v.txt 2>&1
done; done
