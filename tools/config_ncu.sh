#!/bin/bash
# per-kernel time / DRAM / fp64 pipe / SM balance of one decode of a config (second of two decodes)
# usage: tools/config_ncu.sh CODE B ITERS EBNO EARLY PREC > out.csv ; python tools/ncu_by_kernel.py out.csv
ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_active.max,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size \
    --clock-control none --csv python tools/config_profile.py "$@" 1 2>/dev/null
