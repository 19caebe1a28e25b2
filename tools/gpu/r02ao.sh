O=gpurun_out/r02ao; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for v in td11 td15; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so C3 >> $O/variants.txt 2>&1; done
