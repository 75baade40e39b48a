# cache hints x schedule
{
C=$PWD/paper_1609_01567_b200/_native/cached/libldpc_b200.so
for v in "LDPC_TILE=0" "X=1" "LDPC_LIB=$C LDPC_TILE=0" "LDPC_LIB=$C" "LDPC_LIB=$C LDPC_TILE=2"; do
env $v timeout 300 python bench.py --no-e2e --no-cpu --no-fast --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v'[-30:].ljust(30), 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
done
LDPC_LIB=$C timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_(check|node|var)" -s 40 -c 12 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-fast 2>&1 | grep -E "k_|duration|bytes|hit_rate" | head -60
} 2>&1 | tee gpurun_out/tile_probe2.log
