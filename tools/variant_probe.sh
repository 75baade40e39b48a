# env-selected kernel variants, device-timed bench (no e2e/cpu/fast legs); usage: bash tools/variant_probe.sh "ENV=.. ENV2=.." ...
run() {
  env $1 timeout 300 python bench.py --no-e2e --no-cpu --no-fast --no-configs --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1'.ljust(44), 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
}
for v in "$@"; do run "$v"; done
