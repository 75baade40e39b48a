#!/bin/bash
# Capture ncu evidence for the bench workload (run under gpurun, 1 GPU).
#   launches_<tag>.csv       : every kernel launch of one bench step (C3) with its device time
#   prof_<tag>_var/check     : --set full captures of the top kernels (variable rings, check)
#   prof_<tag>_c4            : --set full of the high-degree chains kernels (C4: fp64-pipe bound)
#   prof_<tag>_onchip        : --set full of the on-chip decoder (C1, one frame)
#   prof_<tag>_priors        : --set full of the layout kernel without / with the fused AWGN prior
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
# .ncu-rep files go to REP (default /tmp/ncu: gpurun_out must stay under 64 MiB to come back);
# tools/profile_round.sh summarises them into gpurun_out/
REP=${NCU_REP_DIR:-/tmp/ncu}
mkdir -p $REP
BENCH="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-configs --no-fast"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 200 --csv \
    --log-file $OUT/launches_$TAG.csv $BENCH > $OUT/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(var_reg|node_ring)" -s 3 -c 3 \
    -o $REP/prof_${TAG}_var $BENCH > $OUT/ncu_var_$TAG.log 2>&1
echo "var capture rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_check_reg -s 1 -c 1 \
    -o $REP/prof_${TAG}_check $BENCH > $OUT/ncu_check_$TAG.log 2>&1
echo "check capture rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(check|var)_chains" -s 2 -c 2 \
    -o $REP/prof_${TAG}_c4 python bench.py --config C4 --iters 20 --steps 1 --warmup 0 --no-e2e --no-cpu \
    --no-configs --no-fast > $OUT/ncu_c4_$TAG.log 2>&1
echo "c4 capture rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_onchip -s 0 -c 1 \
    -o $REP/prof_${TAG}_onchip python bench.py --config C1 --batch 1 --iters 50 --steps 1 --warmup 0 --no-e2e \
    --no-cpu --no-configs --no-fast > $OUT/ncu_onchip_$TAG.log 2>&1
echo "onchip capture rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_transpose_priors -s 20 -c 2 \
    -o $REP/prof_${TAG}_priors python tools/prior_kernel_probe.py > $OUT/ncu_priors_$TAG.log 2>&1
echo "priors capture rc=$?"
# round 2: C4 per-kernel fp64-pipe activity and SM balance (metric list, exact and fast mode);
# --set full of the O(d) fast-mode kernels (C4) and of the compaction kernels (C2, early stop)
bash tools/c4_ncu.sh fp64 > $OUT/c4_fp64_$TAG.csv 2> /dev/null
bash tools/c4_ncu.sh fp32 > $OUT/c4_fp32_$TAG.csv 2> /dev/null
echo "c4 metric lists rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(check|var)_f32_od" -s 10 -c 4 \
    -o $REP/prof_${TAG}_fastod python tools/c4_profile.py fp32 1 > $OUT/ncu_fastod_$TAG.log 2>&1
echo "fast O(d) capture rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_compact" -s 4 -c 4 \
    -o $REP/prof_${TAG}_compact python tools/compact_breakdown.py C2 4096 20 2.0 > $OUT/ncu_compact_$TAG.log 2>&1
echo "compaction capture rc=$?"
ls -la $OUT $REP
