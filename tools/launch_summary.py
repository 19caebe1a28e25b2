"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, gzip, sys
rows = [r for r in csv.reader((gzip.open if sys.argv[1].endswith(".gz") else open)(sys.argv[1], "rt")) if len(r) > 5]
hdr, data = rows[0], rows[1:]
iN, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if r[iM] == "gpu__time_duration.sum":
        k = r[iN].split("(")[0][:60]
        agg[k][0] += 1
        agg[k][1] += float(r[iV])
tot = sum(v[1] for v in agg.values())
print(f"# {sys.argv[1]}: {sum(v[0] for v in agg.values())} launches, {tot / 1e6:.2f} ms summed "
      "(cold-cache, serialised under ncu: shares, not absolute step time)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} n={v[0]:5d} total={v[1] / 1e6:8.3f} ms avg={v[1] / v[0] / 1e3:9.2f} us share={v[1] / tot * 100:5.1f}%")
