"""Summarise an ncu report: key metrics, stall mix, opcode mix, top stalls."""
import csv, subprocess, sys, io
rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
d = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
hdr = d[0]
want = ['Duration', 'Registers Per Thread', 'Achieved Occupancy', 'Compute (SM) Throughput', 'DRAM Throughput',
        'Executed Ipc Active', 'Block Size', 'Grid Size', 'Issue Slots Busy', 'Eligible Warps Per Scheduler',
        'Cluster Size', 'Max Active Clusters', 'Waves Per SM', 'Dynamic Shared Memory Per Block']
seen = set()
for row in d[1:]:
    r = dict(zip(hdr, row))
    if kfilter and kfilter not in r['Kernel Name']:
        continue
    k = (r['ID'], r['Metric Name'])
    if r['Metric Name'] in want and k not in seen:
        seen.add(k); print(r['ID'], r['Kernel Name'][:40], '|', r['Metric Name'], r['Metric Value'], r['Metric Unit'])
rows = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
hidx = [i for i, r in enumerate(rows) if r and r[0] == 'Address']
for si, h0 in enumerate(hidx):
    hdr = rows[h0]; data = rows[h0 + 1:(hidx[si + 1] - 1 if si + 1 < len(hidx) else len(rows))]
    iS = hdr.index("Warp Stall Sampling (All Samples)"); iSrc = hdr.index("Source"); iE = hdr.index("Instructions Executed")
    tot = sum(float(r[iS] or 0) for r in data if len(r) > iS)
    agg, ops = {}, {}
    for r in data:
        if len(r) <= iE: continue
        for j, h in enumerate(hdr):
            if h.startswith('stall_') and '(Not' not in h and r[j] not in ('0', ''):
                try: agg[h] = agg.get(h, 0) + float(r[j])
                except ValueError: pass
        toks = r[iSrc].split()
        if toks:
            op = (toks[1] if toks[0].startswith('@') else toks[0]).split('.')[0]
            try: ops[op] = ops.get(op, 0) + float(r[iE] or 0)
            except ValueError: pass
    t2 = sum(ops.values()) or 1
    print(f"section {si}: samples {tot:.0f} insts {t2:.3g}")
    print("  stalls:", [(k[6:], round(v / tot, 3)) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:9]])
    print("  ops:", [(k, round(v / t2, 3)) for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:16]])
