# C5 north-star gate experiment on the box (GPU + threaded oracle on the host cores)
O=gpurun_out/r02b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 1500 python tools/c5_gate_experiment.py 1e-10 1e-12 > $O/c5_gate.txt 2>&1; echo "rc=$?" >> $O/c5_gate.txt
