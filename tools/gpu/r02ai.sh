O=gpurun_out/r02ai; mkdir -p $O
R=/tmp/rep; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:'^k_march$' -c 1 -o $R/march -f python tools/one_solve.py C5 > $O/n1.log 2>&1
$NCU -k regex:'^k_cgs$' --launch-skip 600 -c 1 -o $R/cgs -f python tools/one_solve.py C5 > $O/n3.log 2>&1
$NCU -k regex:'^k_march$' --launch-skip 1 -c 1 -o $R/tdm -f python tools/one_solve.py C3 > $O/n7.log 2>&1
for r in march cgs tdm; do echo "######## $r" >> $O/ncu_brief.txt; python tools/ncu_brief.py $R/$r.ncu-rep >> $O/ncu_brief.txt 2>&1; python tools/ncu_summary.py $R/$r.ncu-rep >> $O/ncu_full_$r.txt 2>&1; done
ncu -i $R/march.ncu-rep --page raw --csv > $O/raw_march.csv 2>/dev/null; gzip -f $O/raw_march.csv
