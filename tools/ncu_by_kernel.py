"""Aggregate an ncu --csv metrics list per kernel (second half of the launches = the measured decode).
usage: python tools/ncu_by_kernel.py file.csv [--all]"""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
rows = rows[1:]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
by_id = collections.OrderedDict()
for r in rows:
    by_id.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", "")) if r[vi] else 0.0
launches = list(by_id.values())
if "--all" not in sys.argv:
    launches = launches[len(launches) // 2:]  # the script decodes twice: keep the second
agg = collections.OrderedDict()
for L in launches:
    name = L["name"].split("(")[0].replace("void ", "").replace("ldpc::", "").replace("<unnamed>::", "")
    a = agg.setdefault(name, collections.defaultdict(float))
    a["n"] += 1
    a["us"] += L.get("gpu__time_duration.sum", 0) / 1e3
    a["fp64_pct_x_us"] += L.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0) * L.get("gpu__time_duration.sum", 0) / 1e3
    a["bal_x_us"] += (L.get("sm__cycles_active.avg", 0) / max(L.get("sm__cycles_active.max", 1), 1)) * L.get("gpu__time_duration.sum", 0) / 1e3
    a["dram_MB"] += (L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)) / 1e6
total = sum(a["us"] for a in agg.values())
out = {}
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
    out[k] = {"launches": int(a["n"]), "us": round(a["us"], 1), "share": round(a["us"] / total, 3),
              "fp64_pipe_pct": round(a["fp64_pct_x_us"] / a["us"], 1) if a["us"] else 0,
              "sm_active_balance": round(a["bal_x_us"] / a["us"], 3) if a["us"] else 0,
              "dram_MB": round(a["dram_MB"], 1)}
print(json.dumps({"total_us": round(total, 1), "kernels": out}, indent=1))
