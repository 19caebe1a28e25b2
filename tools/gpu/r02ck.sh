# e2e overhead breakdown
O=gpurun_out/r02ck; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python tools/e2e_parts.py > $O/parts.txt 2>&1
