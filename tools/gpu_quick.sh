# quick GPU check: parity tests + device-timed bench (no e2e/cpu/fast legs); log in gpurun_out/quick.log
{
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
for k in 1 2; do
timeout 300 python bench.py --no-e2e --no-cpu --no-fast --no-configs --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), 'frac', round(r['frac'],3), 'stepGBps', round(r['step_algorithmic_GBps']), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
done
} 2>&1 | tee gpurun_out/quick.log
