# A/B of the stored b_k on the NL streaming sweep (same box, alternating)
O=gpurun_out/r02cd; mkdir -p $O
for i in 1 2 3; do
  timeout 200 python tools/nl_stream_time.py build_variants/libswr_old.so >> $O/nls.txt 2>&1
  timeout 200 python tools/nl_stream_time.py build_variants/libswr_new.so >> $O/nls.txt 2>&1
done
