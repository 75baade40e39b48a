#!/bin/bash
# A/B of run-time switches on one config (tools/config_profile.py), alternating K times.
# usage: tools/ab_env_config.sh K "CODE B ITERS EBNO EARLY PREC" "ENV=a" "-" ...
K=$1; CFG=$2; shift 2
for k in $(seq 1 $K); do
  for e in "$@"; do
    if [ "$e" = - ]; then envs=""; else envs="$e"; fi
    echo "$e $(env $envs python tools/config_profile.py $CFG 5 | grep -o 'ms per decode [0-9.]*')"
  done
done
