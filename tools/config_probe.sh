# device-timed throughput of the other BASELINE configs, on-chip (auto) vs streaming (LDPC_ONCHIP=0)
{
for v in "X=0" "LDPC_ONCHIP=0"; do
for c in "--config C2 --iters 20" "--config C1 --batch 1 --iters 50" "--config C1 --batch 4096 --iters 50" "--config C4 --iters 20"; do
env $v timeout 600 python bench.py $c --no-e2e --no-cpu --no-fast --steps 5 --warmup 3 2>gpurun_out/cfg.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $c'.ljust(52), 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],4), 'launches/step', d['gpu_launches']/5)" || tail -3 gpurun_out/cfg.err
done; done
} 2>&1 | tee gpurun_out/config_probe.log
