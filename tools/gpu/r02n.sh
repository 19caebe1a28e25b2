# new fixed-order reduce: full GPU suite; ncu of the FFT apply and the reduce
O=gpurun_out/r02n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
R=/tmp/rep; mkdir -p $R
ncu --set full --clock-control none --import-source on -k regex:k_fft_conv_reg --launch-skip 400 -c 1 -o $R/fft -f python tools/one_solve.py C5 > $O/ncu_fft.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cgs_reduce --launch-skip 800 -c 2 -o $R/red -f python tools/one_solve.py C5 > $O/ncu_red.log 2>&1
python tools/ncu_brief.py $R/fft.ncu-rep $R/red.ncu-rep > $O/ncu_brief.txt 2>&1
cp $R/*.ncu-rep $O/
timeout 1800 python -m pytest tests -q -m gpu -rf --durations=5 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
