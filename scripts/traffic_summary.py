"""Summarise ncu captures of scripts/traffic_products.py into profiles/<round>/traffic.json:
per (config, product): DRAM bytes read + written over the product's kernels, one launch each.
    python scripts/traffic_summary.py gpurun_out/traffic_c3.csv ... > profiles/r02/traffic.json"""
import csv
import json
import os
import re
import sys

entries = []
for f in sys.argv[1:]:
    m = re.search(r"traffic_(c\d)_(xv|xtu)", os.path.basename(f))
    cfg, prod = m.group(1), m.group(2)
    hdr = None
    for r in csv.reader(open(f)):
        if r and r[0] == "ID":
            hdr = r
            break
    iname, imet, ival = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    kern = {}
    for r in csv.reader(open(f)):
        if len(r) > ival and r[0].isdigit():
            k = kern.setdefault(int(r[0]), {"name": r[iname], "m": {}})
            k["m"][r[imet]] = float(r[ival].replace(",", ""))
    ks = [kern[i] for i in sorted(kern)]
    rd = sum(k["m"].get("dram__bytes_read.sum", 0) for k in ks)
    wr = sum(k["m"].get("dram__bytes_write.sum", 0) for k in ks)
    ns = sum(k["m"].get("gpu__time_duration.sum", 0) for k in ks)
    names = [re.sub(r"\(.*", "", k["name"]).replace("void ", "").replace("ssa::", "") for k in ks]
    path = "fft" if any("pass" in n for n in names) else ("tc" if any("hankel" in n for n in names) else "direct")
    entries.append({"config": cfg, "product": prod, "path": path, "dram_read_bytes": rd, "dram_write_bytes": wr,
                    "traffic_bytes": rd + wr, "kernel_ns_sum": ns, "kernels": names})
print(json.dumps({"source": "ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                            "gpu__time_duration.sum over the kernels of one block product "
                            "(scripts/traffic_products.py, solver layout, ncu default cache control: cold caches)",
                  "entries": entries}, indent=1))
