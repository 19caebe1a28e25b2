# FFT apply: twiddle loads hoisted above the PDL wait (A/B, C5 interface time)
O=gpurun_out/r02cu; mkdir -p $O
for i in 1 2; do for v in base twpre; do echo "== $v" >> $O/c5.txt; timeout 300 python tools/quick_c5.py C5 build_variants/libswr_$v.so 2>&1 | grep status >> $O/c5.txt; done; done
