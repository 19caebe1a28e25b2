O=gpurun_out/r02e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for v in unitslot unitsub; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so >> $O/variants.txt 2>&1; done
timeout 900 python -m pytest tests/test_multirank.py tests/test_gpu_parity.py -q -k "stream or cgs or multirank or logical or deterministic" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
R=/tmp/rep; mkdir -p $R
ncu --set full --clock-control none --import-source on -k regex:'k_cgs<' --launch-skip 60 -c 1 -o $R/cgs_dots -f python tools/one_solve.py C5 > $O/ncu_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cgs_axpy --launch-skip 60 -c 1 -o $R/cgs_axpy -f python tools/one_solve.py C5 > $O/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fft_conv_reg --launch-skip 30 -c 1 -o $R/fft -f python tools/one_solve.py C5 > $O/ncu_c.log 2>&1
python tools/ncu_brief.py $R/cgs_dots.ncu-rep $R/cgs_axpy.ncu-rep $R/fft.ncu-rep > $O/ncu_summary.txt 2>&1
cp $R/*.ncu-rep $O/ 2>/dev/null
ls -la $O
