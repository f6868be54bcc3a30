mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "linear or float32 or select or golden or extreme" > gpurun_out/r02h_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02h_tests.log
timeout 600 python bench.py --config linear --steps 10 --warmup 3 > gpurun_out/r02h_linear.json 2> gpurun_out/r02h_linear.err
timeout 300 python scripts/exp_select.py > gpurun_out/r02h_select.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:linear|gate' --csv --log-file gpurun_out/r02h_linear_launches.csv python bench.py --config linear --steps 2 --warmup 1 > gpurun_out/r02h_linear_ncu.log 2>&1
tail -3 gpurun_out/r02h_tests.log
