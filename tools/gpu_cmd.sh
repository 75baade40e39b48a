timeout 900 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo bench_rc=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r1.json 2>&1
bash profiles/ncu_capture.sh r1c
python tools/ncu_traffic.py gpurun_out/prof_r1c_var.ncu-rep gpurun_out/prof_r1c_check.ncu-rep gpurun_out/ncu_traffic.json
