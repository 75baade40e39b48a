"""Summarise ncu reports / launch lists into text (what gets committed under profiles/)."""
import collections
import csv
import io
import json
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__bytes_read.sum", "MB", 1e-6),
    ("dram__bytes_write.sum", "MB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%", 1),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "%", 1),
    ("launch__registers_per_thread", "", 1),
    ("launch__occupancy_limit_registers", "", 1),
    ("smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct", "%", 1),
    ("smsp__warps_issue_stalled_lg_throttle_per_warp_active.pct", "%", 1),
    ("smsp__warps_issue_stalled_wait_per_warp_active.pct", "%", 1),
    ("smsp__warps_issue_stalled_math_pipe_throttle_per_warp_active.pct", "%", 1),
    ("smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct", "%", 1),
    ("smsp__warps_issue_stalled_drain_per_warp_active.pct", "%", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "%", 1),
    ("lts__t_sector_hit_rate.pct", "%", 1),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = re.sub(r"\(.*", "", d.get("Kernel Name", "?")).replace("void ", "").replace("(anonymous namespace)::", "")
        e = {"kernel": name.strip(), "grid": d.get("Grid Size"), "block": d.get("Block Size")}
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
        for m, u, sc in METRICS:
            if m in d and d[m] not in ("", "n/a"):
                try:
                    v = float(d[m].replace(",", ""))
                    unit = units[hdr.index(m)]
                    if unit in scale:  # normalise to bytes -> MB, time -> us
                        v = v * scale[unit] * (1e-6 if "byte" in unit else 1)
                    e[m] = round(v, 3)
                except ValueError:
                    pass
        res.append(e)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for d in data:
        k = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("(anonymous namespace)::", "").strip()
        v = float(d["Metric Value"].replace(",", ""))
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "total_us": round(v / 1e3, 1), "share": round(v / s, 4)}
            for k, v in sorted(tot.items(), key=lambda x: -x[1])]


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(report(path) if kind == "rep" else launches(path), indent=1))
