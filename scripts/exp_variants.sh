#!/bin/bash
# run scripts/exp_k2.py against each built variant (EXP_HEADS, EXP_MODES pass through)
for v in "$@"; do
  echo "== $v"
  ROPESLR_LIBRARY=paper_2605_20659_b200/_variants/$v.so EXP_MODES="${EXP_MODES:-0}" timeout 300 python scripts/exp_k2.py 2>&1 | tail -3
done
