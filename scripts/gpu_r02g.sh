mkdir -p gpurun_out
KRE='regex:pool_blocks|block_scores|select_|nonfinite'
EXP_REPS=1 EXP_ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv --log-file gpurun_out/r02g_select_launches.csv python scripts/exp_select.py > gpurun_out/r02g_select_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:linear|gate' --csv --log-file gpurun_out/r02g_linear_launches.csv python bench.py --config linear --steps 2 --warmup 1 > gpurun_out/r02g_linear_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:linear_state|linear_apply' -c 2 -o gpurun_out/r02g_linear_full -f python bench.py --config linear --steps 1 --warmup 1 > gpurun_out/r02g_linear_full.log 2>&1
tail -2 gpurun_out/r02g_linear_full.log
