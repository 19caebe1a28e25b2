O=gpurun_out/r02i; mkdir -p $O
for v in k l m n; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so >> $O/variants.txt 2>&1; done
