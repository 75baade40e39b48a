#!/bin/bash
# Quick A/B of kernel policies on the bench workload (device-timed value + per-class kernel ms).
for cfg in "DEFAULT=1" ${EXTRA_VARIANTS:-}; do
  cfg=${cfg//,/ }
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/v.json')); r=d['roofline']
print('$cfg', 'value=%.3f'%d['value'], 'frac=%.3f'%r['frac'], r['kernel'], {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})" || tail -5 gpurun_out/v.err
done
