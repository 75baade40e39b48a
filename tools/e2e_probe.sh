# e2e (host API) timing vs sub-batch plan growth and compute lanes
{
for v in "X=0" "LDPC_E2E_GROWTH=170" "LDPC_E2E_GROWTH=200" "LDPC_E2E_LANES=1" "LDPC_E2E_LANES=3" "X=1"; do
env $v timeout 300 python bench.py --no-cpu --no-fast --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v'.ljust(30), 'device ms', round(d['ms_per_step'],3), 'e2e ms', round(d['e2e']['ms_per_step'],3), 'e2e Gbit/s', round(d['e2e']['value'],3), 'stream ms', round(d['e2e_stream']['ms_per_step'],3))"
done
} 2>&1 | tee gpurun_out/e2e_probe.log
