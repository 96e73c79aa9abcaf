"""Summarise ncu reports / launch lists into profiles/ (tools/, not product).

    python tools/ncu_summary.py rep gpurun_out/prof.ncu-rep [...]     # --set full captures
    python tools/ncu_summary.py launches gpurun_out/launches.csv       # gpu__time_duration list
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_B",
    "dram__bytes_write.sum": "dram_write_B",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__warps_eligible.avg.per_cycle_active": "eligible_per_sched",
    "smsp__average_warp_latency_per_inst_issued.ratio": "cycles_per_issue",
}
STALL = "smsp__average_warps_issue_stalled_"


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def raw(rep):
    """Per launch: durations in microseconds, DRAM bytes in bytes (each column's unit applied)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")[:80], "id": d.get("ID")}
        for k, v in KEYS.items():
            if k in d:
                try:
                    rec[v] = float(d[k].replace(",", "")) * SCALE.get(units.get(k, ""), 1)
                except ValueError:
                    rec[v] = d[k]
        stalls = {}
        for k, v in d.items():
            if k.startswith(STALL) and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls[k[len(STALL):-len("_per_issue_active.ratio")]] = float(v.replace(",", ""))
                except ValueError:
                    pass
        rec["top_stalls"] = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
        res.append(rec)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": v[0], "avg_us": v[1] / v[0] / 1e3, "share": v[1] / tot}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]


if __name__ == "__main__":
    mode, paths = sys.argv[1], sys.argv[2:]
    for p in paths:
        print(f"## {p}")
        rows = raw(p) if mode == "rep" else launches(p)
        for r in rows:
            print(r)
