# k_factor: zero-pivot test without hypot (A/B through swr_update_inputs of V_x)
O=gpurun_out/r02co; mkdir -p $O
for v in base nohypot base nohypot; do echo "== $v" >> $O/parts.txt; timeout 300 python tools/e2e_parts.py build_variants/libswr_$v.so 2>&1 | grep update >> $O/parts.txt; done
