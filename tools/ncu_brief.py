"""Brief text summary of an ncu report: key metrics, dram bytes, stall and op mix per kernel."""
import csv, io, subprocess, sys


def run(rep, args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Eligible Warps Per Scheduler", "Achieved Occupancy", "Registers Per Thread",
        "Block Size", "Grid Size", "Cluster Size", "Dynamic Shared Memory Per Block", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Waves Per SM"]
for rep in sys.argv[1:]:
    rows = list(csv.reader(io.StringIO(run(rep, ["--page", "details", "--csv"]))))
    hdr = rows[0]
    iI, iK, iM, iV, iU = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    seen = set()
    print(f"## {rep}")
    for r in rows[1:]:
        if r[iM] in WANT and (r[iI], r[iM]) not in seen:
            seen.add((r[iI], r[iM]))
            print(f"  [{r[iI]}] {r[iK][:40]:40s} {r[iM]:34s} {r[iV]} {r[iU]}")
    raw = list(csv.reader(io.StringIO(run(rep, ["--page", "raw", "--csv", "--metrics",
                                                "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"]))))
    if len(raw) > 2:
        h = raw[0]
        for r in raw[2:]:
            d = dict(zip(h, r))
            print(f"  [{d.get('ID')}] dram read {d.get('dram__bytes_read.sum')} {raw[1][h.index('dram__bytes_read.sum')]}, "
                  f"write {d.get('dram__bytes_write.sum')} {raw[1][h.index('dram__bytes_write.sum')]}, "
                  f"time {d.get('gpu__time_duration.sum')} {raw[1][h.index('gpu__time_duration.sum')]}")
