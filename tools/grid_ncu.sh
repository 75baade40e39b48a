#!/bin/bash
# ncu --set full of the grid schedule's cooperative kernel on one C3 frame (decode(y, sigma2)),
# with source-level stall sampling; the report comes back in gpurun_out/ (small: one launch).
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid -s 8 -c 1 \
    -o gpurun_out/grid_c3 -f python tools/latency_probe.py > gpurun_out/grid_ncu.log 2>&1
echo "grid capture rc=$?"
ls -la gpurun_out/grid_c3.ncu-rep
