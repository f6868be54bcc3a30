#!/bin/bash
# Kernel A/B by environment switch: ncu launch times of the kernels matching
# KRE at config 3, once per "NAME=VALUE" setting (or "cur" for none).
#   usage: KRE='regex:block_scores' gpurun -- bash scripts/env_ab.sh cur ROPESLR_SCORES=dmma
mkdir -p gpurun_out
for v in "$@"; do
  tag=$(echo "$v" | tr '=/' '__')
  if [ "$v" = cur ]; then envs=""; else envs="$v"; fi
  env $envs timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "${KRE:-regex:block_scores}" --csv \
    --log-file gpurun_out/envab_$tag.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-rope-pass \
    > /dev/null 2>&1
  echo "$v $(grep -v '^==' gpurun_out/envab_$tag.csv | tail -n +2 | awk -F'","' '{print $5 ":" $NF}' | tr -d '"' | tr '\n' ' ')"
done
