O=gpurun_out/r02ag; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for v in sm2 sm3 sm4; do timeout 300 python tools/variant_c5.py build_variants/libswr_$v.so C2 >> $O/variants.txt 2>&1; done
