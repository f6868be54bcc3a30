#!/bin/bash
# tests + bench + launch list (no full capture)
tag=${1:-q}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/${tag}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${tag}_bench.log
KRE='regex:pool_blocks|block_scores|select_|lowrank|gate_|sparse_attn|key_block_norm|fuse_output|linear_|rope_pool'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" \
  > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}_ncu.log
tail -3 gpurun_out/${tag}_pytest.log; tail -2 gpurun_out/${tag}_bench.log
