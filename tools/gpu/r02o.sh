# warm-cache launch lists (ncu --cache-control none): per-kernel cost inside the flow
O=gpurun_out/r02o; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $O/warm_c5.csv python tools/one_solve.py C5 > $O/ncu_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $O/warm_c4.csv python tools/one_solve.py C4 > $O/ncu_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $O/warm_c3.csv python tools/one_solve.py C3 > $O/ncu_c3.log 2>&1
gzip -f $O/*.csv
