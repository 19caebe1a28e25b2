# stall sampling of one k_fft_conv_reg launch at C5: top source lines
R=/tmp/rep; mkdir -p $R gpurun_out/prof
ncu --set full --import-source on --clock-control none -k regex:k_fft_conv_reg --launch-skip 25 -c 1 -o $R/fftsrc -f \
    python tools/one_solve.py C5 > /dev/null 2>&1
ncu -i $R/fftsrc.ncu-rep --page source --csv --print-source sass > $R/fft_sass.csv 2>/dev/null
ncu -i $R/fftsrc.ncu-rep --page details --csv > $R/fft_details.csv 2>/dev/null
python - <<'PY'
import csv
rows = list(csv.reader(open('/tmp/rep/fft_sass.csv')))
hdr = rows[0]
print(hdr[:12])
def col(name):
    for i, h in enumerate(hdr):
        if h.strip() == name: return i
    return None
iS = col("Warp Stall Sampling (All Samples)")
iSrc = col("Source")
tot = sum(float(r[iS] or 0) for r in rows[1:] if len(r) > iS)
top = sorted(rows[1:], key=lambda r: -float(r[iS] or 0))[:25]
print("total samples", tot)
for r in top:
    print(f"{float(r[iS])/tot*100:5.1f}%  {r[iSrc][:110]}")
PY
grep -i "stall\|warp cycles per issued" /tmp/rep/fft_details.csv | head -30
