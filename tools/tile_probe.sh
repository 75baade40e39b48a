# tiled (L2-resident) vs streaming schedule
{
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
for v in "LDPC_TILE=0" "X=1" "LDPC_TILE=2" "LDPC_TILE_MB=60" "LDPC_TILE_MB=100"; do
env $v timeout 300 python bench.py --no-e2e --no-cpu --no-fast --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v'.ljust(18), 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), 'frac', round(r['frac'],3), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()}, d['gpu_launches'])"
done
} 2>&1 | tee gpurun_out/tile_probe.log
