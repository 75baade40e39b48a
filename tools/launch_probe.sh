# per-kernel device times (ncu launch list, cold-ish, serialized) for env variants
# usage: bash tools/launch_probe.sh "VAR=a VAR2=b" "VAR=c" ...
mkdir -p gpurun_out
i=0
for v in "$@"; do
  i=$((i+1))
  env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
     --log-file gpurun_out/lp_$i.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-fast --no-configs > /dev/null 2>&1
  python - "$v" gpurun_out/lp_$i.csv <<'PY'
import csv, sys, collections, statistics
rows = [r for r in csv.DictReader(l for l in open(sys.argv[2]) if l.startswith('"'))]
t = collections.defaultdict(list)
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("ldpc::<unnamed>::", "")
        t[name + "(" + r["Kernel Name"].split("(")[1].split(")")[0][:0] + ")"].append(float(r["Metric Value"]))
print("==", sys.argv[1])
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    if sum(v) > 50:
        print(f"   {k[:60]:60s} n={len(v):3d} median={statistics.median(v):8.1f} us total={sum(v):9.1f}")
PY
done
