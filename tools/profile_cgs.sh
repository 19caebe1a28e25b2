# --set full captures of the CGS dots pass and update pass at C5 (summaries only)
O=gpurun_out/prof; mkdir -p $O; R=/tmp/rep; mkdir -p $R
ncu --set full --clock-control none --import-source on -k regex:'^k_cgs$' --launch-skip 50 -c 1 -o $R/cgs_dots -f \
    python tools/one_solve.py C5 > $O/ncu_c.log 2>&1
[ -f $R/cgs_axpy.ncu-rep ] || ncu --set full --clock-control none --import-source on -k regex:k_cgs_axpy --launch-skip 50 \
    -c 1 -o $R/cgs_axpy -f python tools/one_solve.py C5 > $O/ncu_d.log 2>&1
python tools/ncu_brief.py $R/cgs_dots.ncu-rep $R/cgs_axpy.ncu-rep > $O/ncu_summary_cgs.txt 2>&1
