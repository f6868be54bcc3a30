timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
for kv in 0.9 0.5; do
python scripts/exp_keep_k1.py $kv
ROPESLR_KEEP_SORT=bitonic python scripts/exp_keep_k1.py $kv
done
ncu --set full --clock-control none --import-source on -k regex:select_keep -s 2 -c 1 -o gpurun_out/keep_new python scripts/exp_keep_k1.py > /dev/null 2>&1
