#!/bin/bash
# Capture ncu evidence for the bench workload (run under gpurun, 1 GPU).
#   launches_<tag>.csv : every kernel launch of one decode step with its device time
#   prof_<tag>_*.ncu-rep : --set full captures of the top kernels
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-configs"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(check|var|node|syndrome|update|transpose|pack|finalize|count|fill)" -c 120 --csv \
    --log-file $OUT/launches_$TAG.csv $BENCH > $OUT/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(var_reg|node_ring)" -s 3 -c 3 \
    -o $OUT/prof_${TAG}_var $BENCH > $OUT/ncu_var_$TAG.log 2>&1
echo "var capture rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_check_reg -s 1 -c 1 \
    -o $OUT/prof_${TAG}_check $BENCH > $OUT/ncu_check_$TAG.log 2>&1
echo "check capture rc=$?"
ls -la $OUT
