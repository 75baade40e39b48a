# high-degree (C4) parity + timing of the wide check kernel variants
{
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "C4 or wide or cli or phases or edge" 2>&1 | tail -2
for v in "X=0" "LDPC_CHAIN_R=8"; do
env $v timeout 600 python bench.py --config C4 --iters 20 --no-e2e --no-cpu --no-fast --steps 5 --warmup 3 2>gpurun_out/cfg.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v'.ljust(18), 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/cfg.err
done
} 2>&1 | tee gpurun_out/c4_probe.log
