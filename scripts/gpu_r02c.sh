mkdir -p gpurun_out
KRE='regex:pool_blocks|block_scores|select_|nonfinite'
EXP_REPS=1 EXP_ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv --log-file gpurun_out/r02c_select_launches.csv python scripts/exp_select.py > gpurun_out/r02c_select_ncu.log 2>&1
EXP_REPS=1 EXP_ITERS=1 timeout 900 ncu --set full --clock-control none -k 'regex:select_topk' -c 2 -o gpurun_out/r02c_select_full -f python scripts/exp_select.py > gpurun_out/r02c_select_full.log 2>&1
tail -2 gpurun_out/r02c_select_ncu.log
