#!/bin/bash
# A/B of library builds on the C3 bench step (device-timed, no e2e/cpu/fast/config legs), alternating
# builds K times.  usage: tools/ab_bench.sh K lib1 lib2 ...   ("default" = the in-tree build)
K=$1; shift
for k in $(seq 1 $K); do
  for lib in "$@"; do
    if [ "$lib" = default ]; then unset LDPC_LIB; else export LDPC_LIB=$lib; fi
    timeout 300 python bench.py --no-e2e --no-cpu --no-fast --no-configs --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$lib', 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), 'var frac', round(r['class_frac']['variable'],3), 'check frac', round(r['class_frac']['check'],3), 'sm', d['clocks'].get('sm_mhz'), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
  done
done
