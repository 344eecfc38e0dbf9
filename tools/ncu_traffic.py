"""Write profiles/ncu_traffic.json: {tag: dram__bytes_read.sum + dram__bytes_write.sum per launch} from
`ncu --page raw --csv` exports of single-kernel `--set full` captures.
Usage: python tools/ncu_traffic.py TAG=gpurun_out/raw_X.csv [TAG=...]"""
import csv
import json
import os
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out_p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
res = json.load(open(out_p)) if os.path.exists(out_p) else {}
for arg in sys.argv[1:]:
    tag, path = arg.split("=", 1)
    rows = list(csv.reader(open(path)))
    h, units, vals = rows[0], rows[1], rows[2]
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        tot += float(vals[i].replace(",", "")) * UNITS.get(units[i], 1)
    res[tag] = int(tot)
    print(tag, int(tot), vals[h.index("Kernel Name")][:80])
json.dump(res, open(out_p, "w"), indent=1)
