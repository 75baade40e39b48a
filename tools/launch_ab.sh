#!/bin/bash
# per-kernel device time (ncu launch list of one C3 bench step) for run-time switch variants
# usage: tools/launch_ab.sh "ENV=a" "-" ...
for e in "$@"; do
  if [ "$e" = - ]; then envs=""; else envs="$e"; fi
  echo "== $e"
  env $envs ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_node_ring|k_check_reg" --csv \
      python bench.py --no-e2e --no-cpu --no-fast --no-configs --steps 1 --warmup 1 2>/dev/null \
    | python -c "
import sys, csv, collections
rows = list(csv.reader(sys.stdin))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; rows = [r for r in rows[hi:] if len(r) == len(h)]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
t = collections.defaultdict(list)
for r in rows[1:]:
    t[r[ki].split('(')[0].replace('void ', '')[-40:]].append(float(r[vi].replace(',', '')) / 1e3)
for k, v in sorted(t.items()): print(f'  {k:40s} n={len(v):3d} mean {sum(v)/len(v):7.1f} us')
"
done
