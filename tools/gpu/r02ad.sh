O=gpurun_out/r02ad; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for i in 1 2 3; do timeout 900 python -m pytest tests/test_multirank.py -q -k "precond-vtx" -rf > $O/mr_$i.txt 2>&1; echo "rc=$?" >> $O/mr_$i.txt; done
git stash > /dev/null 2>&1 || true
