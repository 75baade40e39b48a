#!/bin/bash
# A/B of run-time switches on the C3 bench step (device-timed, no e2e/cpu/fast/config legs), alternating
# K times.  usage: tools/ab_env.sh K "ENV=a" "ENV=b" ...   ("-" = no extra environment)
K=$1; shift
for k in $(seq 1 $K); do
  for e in "$@"; do
    if [ "$e" = - ]; then envs=""; else envs="$e"; fi
    env $envs timeout 300 python bench.py --no-e2e --no-cpu --no-fast --no-configs --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$e', 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), 'var frac', round(r['class_frac']['variable'],3), 'check frac', round(r['class_frac']['check'],3), 'sm', d['clocks'].get('sm_mhz'), 'parity', (d.get('parity') or {}).get('mismatches'), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
  done
done
