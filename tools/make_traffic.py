"""profiles/traffic_<cfg>.json from an ncu --set full report (tools/, measurement).

    python tools/make_traffic.py report.ncu-rep C2

DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch, averaged over the
captured launches of each kernel instantiation (e.g. "k_step1_rs<24, 1>").  bench.py reports the
entry of the dominant kernel's instantiation at the profiled inner step as roofline.traffic."""
import csv
import io
import json
import os
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
acc = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "")
    SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    try:  # each column has its own unit (second header row)
        rd = float(d["dram__bytes_read.sum"].replace(",", "")) * SC.get(rows[1][hdr.index("dram__bytes_read.sum")], 1)
        wr = float(d["dram__bytes_write.sum"].replace(",", "")) * SC.get(rows[1][hdr.index("dram__bytes_write.sum")], 1)
    except (KeyError, ValueError):
        continue
    key = name.replace("void ", "").split("(")[0]
    if rd < 1e6:  # gated no-op launches
        continue
    acc.setdefault(key, []).append(rd + wr)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"traffic_{cfg}.json")
# merge: instantiations this capture did not see keep their earlier entries
res = json.load(open(path)) if os.path.exists(path) else {}
prev_src = res.pop("source", "")
res.update({k: sum(v) / len(v) for k, v in acc.items()})
src = f"ncu --set full (cold cache) of bench.py --config {cfg}; DRAM read+write bytes per launch, " \
    "averaged over the captured launches of each kernel instantiation: " + ", ".join(f"{k}:{len(v)}" for k, v in acc.items())
res["source"] = src if not prev_src else prev_src + " | " + src
json.dump(res, open(path, "w"), indent=1)
print(path, res)
