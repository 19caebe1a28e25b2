O=gpurun_out/r02bb; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for v in s1 s3; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so C2 >> $O/variants.txt 2>&1; done
