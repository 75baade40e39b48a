# Round evidence: full bench line, ncu launch list of one step, ncu --set full of the top kernels.
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; tail -c 400 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference_$TAG.json 2> gpurun_out/bench_reference_$TAG.err
echo "reference rc=$?"; tail -c 300 gpurun_out/bench_reference_$TAG.json
bash profiles/ncu_capture.sh $TAG
