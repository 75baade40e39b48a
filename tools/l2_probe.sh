# L2-residency probe: step algorithmic GB/s vs working-set size (C2 code small enough to fit L2)
for B in 64 128 192 256 512 1024 4096; do
  timeout 300 python bench.py --config C2 --iters 10 --batch $B --no-e2e --no-cpu --no-fast --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C2 B=$B', 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), 'stepGBps', round(r['step_algorithmic_GBps']), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()}, 'launches', d['gpu_launches'])"
done
for B in 64 256; do
  timeout 300 python bench.py --config C3 --batch $B --no-e2e --no-cpu --no-fast --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C3 B=$B', 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), 'stepGBps', round(r['step_algorithmic_GBps']), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
done
