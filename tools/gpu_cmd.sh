python tools/fp32_tolerance.py > gpurun_out/fp32_tol.json 2>&1; cat gpurun_out/fp32_tol.json | tail -80
for prec in fp32; do
timeout 600 python -c "
import sys; sys.argv=['bench.py','--steps','10','--warmup','3','--no-cpu','--no-e2e']
" ; done
