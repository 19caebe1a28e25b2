O=gpurun_out/r02be; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $O/c4x.csv python tools/one_solve.py C4 pinv_exact=1 > $O/n.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $O/c3x.csv python tools/one_solve.py C3 pinv_exact=1 > $O/n3.log 2>&1
gzip -f $O/*.csv
