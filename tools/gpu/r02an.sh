# k_march_td: on-chip Re E, z in registers, 9-CTA clusters at C3
O=gpurun_out/r02an; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python tools/quick_c5.py C3 > $O/quick_c3.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py tests/test_race_stress.py -q -k "vtx or precond or C3 or race or solver or pinv" -rf --durations=5 > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
