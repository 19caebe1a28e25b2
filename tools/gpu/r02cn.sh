# refreshed ncu --set full summaries of the kernels changed in round 2's later sessions:
# FFT apply (255 registers), two-pass streaming march (interleaved, 4 per SM, b_k stored),
# NL streaming march, exact causal P^-1 (staged near kernel, far kernel)
O=gpurun_out/r02cn; mkdir -p $O
R=/tmp/rep; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_fft_conv_reg --launch-skip 400 -c 1 -o $R/fft -f python tools/one_solve.py C5 > $O/n1.log 2>&1
$NCU -k regex:k_march_stream2 -c 1 -o $R/stream2 -f python tools/one_solve.py C2 > $O/n2.log 2>&1
$NCU -k regex:k_march_nl_stream -c 1 -o $R/nlstream -f python tools/nl_stream_time.py > $O/n3.log 2>&1
$NCU -k regex:k_pinv_near --launch-skip 20 -c 1 -o $R/pinv_near -f python tools/one_solve.py C4 pinv_exact=1 > $O/n4.log 2>&1
$NCU -k regex:k_pinv_far --launch-skip 20 -c 1 -o $R/pinv_far -f python tools/one_solve.py C4 pinv_exact=1 > $O/n5.log 2>&1
for r in fft stream2 nlstream pinv_near pinv_far; do echo "######## $r" >> $O/ncu_brief.txt; python tools/ncu_brief.py $R/$r.ncu-rep >> $O/ncu_brief.txt 2>&1; python tools/ncu_summary.py $R/$r.ncu-rep >> $O/ncu_full_$r.txt 2>&1; done
ls -la $O
