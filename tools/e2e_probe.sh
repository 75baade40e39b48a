# e2e (host API) timing vs compute lanes and sub-batch plan
{
timeout 600 python -m pytest tests/test_decode_gpu.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -2
for lanes in 1 2; do for sb in 0 256; do
LDPC_E2E_LANES=$lanes timeout 300 python bench.py --no-cpu --no-fast --steps 10 --warmup 3 --sub-batch $sb 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('lanes $lanes sub $sb', 'device ms', round(d['ms_per_step'],3), 'e2e ms', round(d['e2e']['ms_per_step'],3), 'e2e Gbit/s', round(d['e2e']['value'],3))"
done; done
} 2>&1 | tee gpurun_out/e2e_probe.log
