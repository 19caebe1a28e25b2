O=gpurun_out/r02ay; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for v in fb5 fb4; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so C5 >> $O/variants.txt 2>&1; done
for v in fb5 fb4; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so C4 >> $O/variants.txt 2>&1; done
