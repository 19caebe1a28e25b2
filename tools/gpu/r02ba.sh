O=gpurun_out/r02ba; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for v in cg3 cg5 ax3 ax6; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so C5 >> $O/variants.txt 2>&1; done
