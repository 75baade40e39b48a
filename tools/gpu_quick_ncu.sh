bash tools/gpu_quick.sh
TAG=${1:-r1c}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(var_reg|node_ring)" -s 3 -c 3 \
    -o gpurun_out/prof_${TAG}_var python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-fast > gpurun_out/ncu_var_$TAG.log 2>&1
echo "var capture rc=$?"
