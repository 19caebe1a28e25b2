# robustness sweep against the oracle (odd N_j, long N_T, Robin) on the final head
O=gpurun_out/r02ct; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python tools/robustness_check.py > $O/rob.txt 2>&1; echo "rc=$?" >> $O/rob.txt
