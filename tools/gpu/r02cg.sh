# experiment: staggered base addresses of the streaming scratch arrays
O=gpurun_out/r02cg; mkdir -p $O
for i in 1 2; do
  for v in base sk96 sk1296; do
    echo "== $v" >> $O/c2.txt; timeout 300 python tools/quick_c5.py C2 build_variants/libswr_$v.so 2>&1 | grep status >> $O/c2.txt
    timeout 200 python tools/nl_stream_time.py build_variants/libswr_$v.so >> $O/nls.txt 2>&1
  done
done
