"""DRAM traffic per kernel class from an `ncu --set full` capture of one decode phase.

Writes profiles/ncu_traffic.json: for each class (check / variable), the summed
dram__bytes_read.sum + dram__bytes_write.sum of the kernels of one launch group
(all degree buckets of one phase), i.e. per launch as bench.py's roofline counts it.
Usage: python tools/ncu_traffic.py <var.ncu-rep> <check.ncu-rep> [out.json]
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def dram_bytes(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    ir, iw, it = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("gpu__time_duration.sum")
    res = []
    for r in rows[2:]:
        b = float(r[ir]) * SCALE[u[ir]] + float(r[iw]) * SCALE[u[iw]]
        res.append({"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", ""), "dram_bytes": b,
                    "time_us": float(r[it]) * (1e-3 if u[it] == "nsecond" else 1)})
    return res


if __name__ == "__main__":
    var, chk = dram_bytes(sys.argv[1]), dram_bytes(sys.argv[2])
    out = {
        "variable": {"dram_bytes_per_launch": sum(k["dram_bytes"] for k in var), "kernels": var},
        "check": {"dram_bytes_per_launch": sum(k["dram_bytes"] for k in chk), "kernels": chk},
        "source": "ncu --set full --clock-control none (profiles/ncu_capture.sh)",
    }
    path = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json"
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps({k: v["dram_bytes_per_launch"] for k, v in out.items() if isinstance(v, dict)}))
