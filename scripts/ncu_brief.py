"""Key ncu metrics per kernel of a report: python scripts/ncu_brief.py rep.ncu-rep"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
iK, iID, iM, iV, iU = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Executed Instructions",
        "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction", "L2 Hit Rate"]
cur = None; vals = {}
def flush():
    if cur is not None:
        print(f"{cur[0]:>3} {cur[1][:34]:34s} " + "  ".join(f"{k.split()[0][:8]}={vals.get(k, '?')}" for k in want))
for r in rows[1:]:
    if (r[iID], r[iK]) != cur:
        flush(); cur = (r[iID], r[iK]); vals = {}
    if r[iM] in want and r[iM] not in vals:
        vals[r[iM]] = r[iV] + ("" if r[iU] in ("", "%") else r[iU][:2])
flush()
