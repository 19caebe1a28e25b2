# experiment: 17 rows per thread (2-CTA clusters) -- the chooser rejected it (258 KB of shared memory), so both libraries ran the 11-row shape; see DESIGN.md section 6
O=gpurun_out/r02ch; mkdir -p $O
for i in 1 2; do
  for v in base m17; do
    echo "== $v" >> $O/c5.txt; SWR_VERBOSE=1 timeout 300 python tools/quick_c5.py C5 build_variants/libswr_$v.so >> $O/c5.txt 2>&1
  done
done
