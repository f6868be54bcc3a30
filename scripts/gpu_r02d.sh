mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02d_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02d_tests.log
timeout 300 python scripts/exp_select.py > gpurun_out/r02d_select.log 2>&1
KRE='regex:pool_blocks|block_scores|select_|nonfinite'
EXP_REPS=1 EXP_ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv --log-file gpurun_out/r02d_select_launches.csv python scripts/exp_select.py > gpurun_out/r02d_select_ncu.log 2>&1
tail -3 gpurun_out/r02d_tests.log
