# on-chip vs streaming at small batches (calibrates the auto schedule)
{
for c in "C1 1 50" "C1 64 50" "C1 296 50" "C1 592 50" "C2 1 20" "C2 16 20" "C2 74 20" "C2 148 20"; do
set -- $c
for v in "X=0" "LDPC_ONCHIP=0"; do
env $v timeout 600 python bench.py --config $1 --batch $2 --iters $3 --no-e2e --no-cpu --no-fast --steps 10 --warmup 3 2>gpurun_out/cfg.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $c'.ljust(30), 'ms', round(d['ms_per_step'],3))" || tail -3 gpurun_out/cfg.err
done; done
} 2>&1 | tee gpurun_out/config_probe2.log
