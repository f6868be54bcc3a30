timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dit.py tests/test_gpu_host.py tests/test_gpu_keep_select.py -x -q 2>&1 | tail -4
for o in 1 0; do
  ROPESLR_PAIRS64=$o python bench.py --config cfg2_sweep --steps 10 --warmup 3 2>/dev/null | head -3 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('pairs64=$o', d['config']['workload'][-8:], round(d['sparse_branch']['ms'],4), round(d['sparse_branch']['frac_of_bf16_peak'],3))"
  ROPESLR_PAIRS64=$o python bench.py --config cfg4 --steps 3 --warmup 2 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.readline()); print('pairs64=$o cfg4', round(d['ms_per_step'],2))"
done
