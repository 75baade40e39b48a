# Round evidence: full bench line, ncu launch list of one step, ncu --set full of the top kernels.
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; tail -c 400 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference_$TAG.json 2> gpurun_out/bench_reference_$TAG.err
echo "reference rc=$?"; tail -c 300 gpurun_out/bench_reference_$TAG.json
bash profiles/ncu_capture.sh $TAG

# summaries of the captures (the .ncu-rep files stay on the box)
REP=${NCU_REP_DIR:-/tmp/ncu}
for k in var check c4 onchip priors fastod compact; do
  [ -f $REP/prof_${TAG}_$k.ncu-rep ] && python tools/ncu_summary.py rep $REP/prof_${TAG}_$k.ncu-rep > gpurun_out/ncu_${k}_$TAG.json
done
python tools/ncu_summary.py launches gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.json
python tools/ncu_traffic.py $REP/prof_${TAG}_var.ncu-rep $REP/prof_${TAG}_check.ncu-rep gpurun_out/ncu_traffic_$TAG.json
for p in fp64 fp32; do python tools/ncu_by_kernel.py gpurun_out/c4_${p}_$TAG.csv > gpurun_out/c4_${p}_$TAG.json; done
du -sh gpurun_out
