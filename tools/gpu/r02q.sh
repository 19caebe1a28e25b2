O=gpurun_out/r02q; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_fft_conv_reg --launch-skip 20 -c 1 -o $O/fft_n100 -f python tools/fft_probe.py N100 30 > $O/l1.txt 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_fft_conv_reg --launch-skip 20 -c 1 -o $O/fft_c5 -f python tools/fft_probe.py C5 30 > $O/l2.txt 2>&1
