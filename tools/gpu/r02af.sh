O=gpurun_out/r02af; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
SWR_VERBOSE=1 timeout 300 python tools/one_solve.py C2 > $O/one.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_march_stream2 -c 1 -o $O/stream2 -f python tools/one_solve.py C2 > $O/ncu.log 2>&1
