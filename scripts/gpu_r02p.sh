mkdir -p gpurun_out
rm -rf gpurun_out/parity
timeout 900 python -m pytest tests/test_gpu_screen.py -q -x -p no:cacheprovider > gpurun_out/r02p_screen.log 2>&1
echo "exit $?" >> gpurun_out/r02p_screen.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "selection or fullsize or golden or parity or smoke or select" > gpurun_out/r02p_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02p_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02p_bench.json 2> gpurun_out/r02p_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:screen|pool_blocks|select|scores" --csv --log-file gpurun_out/r02p_k1_launches.csv python bench.py --steps 1 --warmup 1 > /dev/null 2>&1
tail -3 gpurun_out/r02p_screen.log gpurun_out/r02p_tests.log
