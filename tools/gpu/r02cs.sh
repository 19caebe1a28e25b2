# bench contract tests (product arm on C1)
O=gpurun_out/r02cs; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 python -m pytest tests/test_bench_contract.py -q -rf > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
