timeout 600 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -x 2>&1 | tail -2
for g in 1 0; do
LDPC_GRAPHS=$g timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/g_$g.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/g_$g.json')); print('graphs=$g', 'value=%.3f'%d['value'], 'e2e=%.3f'%d['e2e']['value'], 'e2e_ms=%.2f'%d['e2e']['ms_per_step'], 'launches', d['gpu_launches'])"
done
for b in 128 256; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --batch $b > gpurun_out/b_$b.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b_$b.json')); print('batch=$b', 'value=%.3f'%d['value'], 'ms=%.2f'%d['ms_per_step'])"
done
