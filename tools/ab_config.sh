#!/bin/bash
# A/B of library builds on one config (tools/config_profile.py), alternating K times.
# usage: tools/ab_config.sh K "CODE B ITERS EBNO EARLY PREC" lib1 lib2 ...  ("default" = in-tree)
K=$1; CFG=$2; shift 2
for k in $(seq 1 $K); do
  for lib in "$@"; do
    if [ "$lib" = default ]; then unset LDPC_LIB; else export LDPC_LIB=$lib; fi
    echo "$lib $(python tools/config_profile.py $CFG 5 | grep -o 'ms per decode [0-9.]*')"
  done
done
