# A/B/C of the stored b_k: old (none), new (both streaming kernels), mix (two-pass linear only)
O=gpurun_out/r02ce; mkdir -p $O
for i in 1 2; do
  for v in old new mix; do
    timeout 200 python tools/nl_stream_time.py build_variants/libswr_$v.so >> $O/nls.txt 2>&1
    echo "== $v" >> $O/c2.txt; timeout 300 python tools/quick_c5.py C2 build_variants/libswr_$v.so 2>&1 | grep status >> $O/c2.txt
  done
done
