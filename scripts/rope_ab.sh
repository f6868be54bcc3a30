#!/bin/bash
# RoPE + pooling pre-pass: parity tests, then its launch time at config 3 for
# the in-tree build, the row-bulk-copy kernel (ROPESLR_ROPE_TMA=0) and any
# variants built with build_variant.sh.
#   usage: gpurun -- bash scripts/rope_ab.sh [variant ...]
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_rope_pool.py -x -q 2>&1 | tail -3
for v in cur tma0 "$@"; do
  unset ROPESLR_LIBRARY ROPESLR_ROPE_TMA
  if [ $v = tma0 ]; then export ROPESLR_ROPE_TMA=0; elif [ $v != cur ]; then
    export ROPESLR_LIBRARY=paper_2605_20659_b200/_variants/$v.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:rope_pool" --csv \
    --log-file gpurun_out/rope_ab_$v.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "$v $(grep rope_pool gpurun_out/rope_ab_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
