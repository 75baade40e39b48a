# A/B of the layout chunk width (LDPC_CHUNK_LOG2 builds under _native/cN)
for L in "" c7 c8; do
  lib=paper_1609_01567_b200/_native/$L/libldpc_b200.so
  for k in 1 2; do
  LDPC_LIB=$PWD/$lib timeout 300 python bench.py --no-e2e --no-cpu --no-fast --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('lib=$L', 'ms', round(d['ms_per_step'],3), 'Gbit/s', round(d['value'],3), 'stepGBps', round(r['step_algorithmic_GBps']), {k: round(v,3) for k,v in r['kernel_ms_per_step'].items()})"
  done
done
LDPC_LIB=$PWD/paper_1609_01567_b200/_native/c8/libldpc_b200.so timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_phases_gpu.py -q -m gpu -x 2>&1 | tail -2
