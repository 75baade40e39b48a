#!/bin/bash
# per-kernel time, fp64-pipe activity and SM-active balance of one C4 decode (after one warm-up decode)
# usage: tools/c4_ncu.sh fp64|fp32 > out.csv
ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_active.max,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size \
    --clock-control none --csv --launch-skip-before-match 0 python tools/c4_profile.py ${1:-fp64} 1 2>/dev/null
