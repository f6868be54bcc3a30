#!/bin/bash
# ncu evidence for the bench command: launch list of our kernels (timing
# pass) and one --set full capture per kernel of the step.
# usage: gpurun --timeout 1800 -- bash scripts/gpu_profile.sh [tag] [bench args...]
tag=${1:-prof}; shift
mkdir -p gpurun_out
KRE=${KRE:-'regex:pool_blocks|block_scores|select_|lowrank|gate_|schedule_units|sparse_attn|key_block_norm|fuse_output|linear_|rope_pool'}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline "$@" \
  > gpurun_out/${tag}_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/${tag}_launches.log
timeout 1200 ncu --set full --clock-control none --import-source on -k "$KRE" -c ${NCU_COUNT:-8} \
  -o gpurun_out/${tag}_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" \
  > gpurun_out/${tag}_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${tag}_full.log
tail -n 2 gpurun_out/${tag}_launches.log; tail -n 2 gpurun_out/${tag}_full.log
