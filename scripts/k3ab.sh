#!/bin/bash
# K3 A/B: ncu launch times of lowrank_umma_kernel at config 3 for the in-tree
# build ("cur") and variants built with build_variant.sh.
#   usage: gpurun -- bash scripts/k3ab.sh <variant> ...
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_compensator.py -x -q 2>&1 | tail -1
for v in cur "$@"; do
  if [ $v = cur ]; then unset ROPESLR_LIBRARY; else export ROPESLR_LIBRARY=paper_2605_20659_b200/_variants/$v.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:lowrank_umma_kernel" --csv \
    --log-file gpurun_out/k3ab_$v.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-rope-pass \
    > /dev/null 2>&1
  echo "$v $(grep lowrank_umma_kernel gpurun_out/k3ab_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
