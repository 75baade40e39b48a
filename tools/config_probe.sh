# device-timed throughput of the other BASELINE configs (C2: batch 4096 x 20 iterations; C4: high degree)
{
timeout 900 python -m pytest tests/test_cli.py tests/test_decode_gpu.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -2
for c in "--config C2 --iters 20" "--config C4 --iters 20" "--config C1 --batch 64 --iters 50"; do
timeout 600 python bench.py $c --no-e2e --no-cpu --no-fast --steps 5 --warmup 3 2>gpurun_out/cfg.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c'.ljust(36), 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), 'frac', round(r['frac'],3), r['kernel'], {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/cfg.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/lp_c4.csv python bench.py --config C4 --iters 20 --steps 1 --warmup 0 --no-e2e --no-cpu --no-fast > /dev/null 2>&1
} 2>&1 | tee gpurun_out/config_probe.log
