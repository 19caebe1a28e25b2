# reference arm line (CPU oracle on the box's cores)
O=gpurun_out/r02cr; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; echo "rc=$?" >> $O/ref.err
