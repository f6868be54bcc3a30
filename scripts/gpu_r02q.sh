mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_screen.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/r02q_screen.log 2>&1
echo "exit $?" >> gpurun_out/r02q_screen.log
timeout 600 python scripts/exp_screen.py > gpurun_out/r02q_exp.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:screen|pool_blocks" --csv --log-file gpurun_out/r02q_k1_launches.csv python scripts/exp_screen.py > /dev/null 2>&1
