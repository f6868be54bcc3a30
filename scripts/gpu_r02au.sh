mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stage1.py -q -x -p no:cacheprovider > gpurun_out/r02au_stage1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:screen_scores|screen_select|pool_blocks_bulk" -c 3 -o gpurun_out/r02au_k1_full -f python bench.py --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:linear_state|linear_apply|linear_gate" -c 3 -o gpurun_out/r02au_linear_full -f python bench.py --config linear --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:stage1_rows|stage1_gram|rows_kernel|xgrad|pre_kernel" -c 8 -o gpurun_out/r02au_train_full -f python bench.py --config train --steps 1 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02au_train_launches.csv python bench.py --config train --steps 2 --warmup 1 > /dev/null 2>&1
