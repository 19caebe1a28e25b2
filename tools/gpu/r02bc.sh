O=gpurun_out/r02bc; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/variant_c5.py build_variants/libswr_s4.so C2 >> $O/variants.txt 2>&1
for v in n3 n4; do timeout 300 python tools/nl_stream_time.py build_variants/libswr_$v.so >> $O/variants.txt 2>&1; done
timeout 300 python tools/nl_stream_time.py >> $O/variants.txt 2>&1
