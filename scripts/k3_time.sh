#!/bin/bash
# K3 / K1 launch times at config 3 (ncu launch list), after the K3 tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_compensator.py tests/test_gpu_stage1.py -x -q 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:lowrank|pool_blocks|block_scores|select_" --csv \
  --log-file gpurun_out/k3_launch.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-rope-pass > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/k3_launch.csv')))
for i, r in enumerate(rows):
    if 'Kernel Name' in r:
        hdr, start = r, i
        break
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
for r in rows[start + 1:]:
    if len(r) > vi:
        print(f"{r[ki].split('(')[0][:60]:60s} {r[vi]:>10s}")
PY
