O=gpurun_out/r02f; mkdir -p $O
(cd build_variants/r1_tree && timeout 300 python tools/quick_c5.py C5 > ../../$O/r1_quick.txt 2>&1)
for v in a b c; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so >> $O/variants.txt 2>&1; done
R=/tmp/rep; mkdir -p $R
ncu --set full --clock-control none --import-source on -k regex:'^k_cgs$' --launch-skip 900 -c 1 -o $R/cgs_dots -f python tools/one_solve.py C5 > $O/ncu_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cgs_axpy --launch-skip 900 -c 1 -o $R/cgs_axpy -f python tools/one_solve.py C5 > $O/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fft_conv_reg --launch-skip 400 -c 1 -o $R/fft -f python tools/one_solve.py C5 > $O/ncu_c.log 2>&1
cp $R/*.ncu-rep $O/ 2>/dev/null
ls -la $O
