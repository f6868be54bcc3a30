mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compensator.py tests/test_gpu_screen.py tests/test_gpu_parity.py tests/test_gpu_host.py tests/test_op.py -q -x -p no:cacheprovider > gpurun_out/r02aa_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02aa_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02aa_bench.json 2> gpurun_out/r02aa_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r02aa_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
