"""Top SASS lines by warp-stall samples of one kernel in an ncu report (tools/, not product).
    python tools/ncu_source_top.py report.ncu-rep [kernel-regex] [N]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else "."
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
blocks = re.split(r'(?m)^"Kernel Name",', out)
for b in blocks[1:]:
    name = b.splitlines()[0]
    if not re.search(pat, name):
        continue
    rows = list(csv.reader(io.StringIO("\n".join(b.splitlines()[1:]))))
    hdr, data = rows[0], rows[1:]
    i_src = hdr.index("Source")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    tot = sum(float(r[i_s] or 0) for r in data if len(r) > i_s)
    print(f"## {name[:100]} samples={tot:.0f}")
    for r in sorted([r for r in data if len(r) > i_s], key=lambda r: -float(r[i_s] or 0))[:N]:
        print(f"{float(r[i_s] or 0):7.0f} {r[i_e]:>8} {r[i_src][:100]}")
