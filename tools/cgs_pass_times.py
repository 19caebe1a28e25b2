"""Per-pass CGS kernel times by Krylov size from a warm ncu launch list."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
data = [r for r in rows[1:] if r[hdr.index('Metric Name')] == 'gpu__time_duration.sum']
iN, iV = hdr.index('Kernel Name'), hdr.index('Metric Value')
seq = [(r[iN].split('(')[0], float(r[iV]) / 1e3) for r in data]
p1, p2, it, i = {}, {}, 0, 0
while i < len(seq) - 2:
    if seq[i][0] == 'k_fft_conv_reg' and 'k_cgs' in seq[i + 1][0] and 'k_cgs' in seq[i + 2][0]:
        p1.setdefault(it % 30, []).append(seq[i + 1][1]); p2.setdefault(it % 30, []).append(seq[i + 2][1])
        it += 1; i += 3
    else:
        if seq[i][0] == 'k_sub': it = 0
        i += 1
tot1 = tot2 = 0
for k in sorted(p1):
    a, b = sum(p1[k]) / len(p1[k]), sum(p2[k]) / len(p2[k]); nv = k + 1
    tot1 += sum(p1[k]); tot2 += sum(p2[k])
    print(f"k={k:2d} pass1 {a:6.2f}us {(nv+1)*8.0/a:5.2f}TB/s  pass2 {b:6.2f}us {(nv+2)*8.0/b:5.2f}TB/s")
print(f"total pass1 {tot1/1e3:.2f} ms pass2 {tot2/1e3:.2f} ms")
