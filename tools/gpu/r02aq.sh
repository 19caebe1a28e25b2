O=gpurun_out/r02aq; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/variant_c5.py build_variants/libswr_mbt.so C5 >> $O/variants.txt 2>&1
timeout 300 python tools/variant_c5.py build_variants/libswr_mbt.so C3 >> $O/variants.txt 2>&1
timeout 300 python tools/variant_c5.py build_variants/libswr_mbt.so C4 >> $O/variants.txt 2>&1
