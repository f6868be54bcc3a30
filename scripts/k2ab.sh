#!/bin/bash
# K2 A/B: parity tests of the in-tree build, then exp_k2 timing of the
# in-tree build ("cur") against kernel variants built with build_variant.sh.
#   usage: gpurun -- bash scripts/k2ab.sh <tag> [variant ...]
tag=${1:-ab}; shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
for rep in 1 2; do
  for v in cur "$@"; do
    if [ $v = cur ]; then unset ROPESLR_LIBRARY; else export ROPESLR_LIBRARY=paper_2605_20659_b200/_variants/$v.so; fi
    echo "== $v" >> gpurun_out/${tag}_ab.log
    EXP_HEADS=${EXP_HEADS:-8} EXP_MODES=0 timeout 300 python scripts/exp_k2.py 2>&1 | grep -v "warm\|ready\|done" >> gpurun_out/${tag}_ab.log
  done
done
tail -3 gpurun_out/${tag}_pytest.log; cat gpurun_out/${tag}_ab.log
