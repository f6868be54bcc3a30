set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02b_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02b_tests.log
timeout 300 python scripts/exp_select.py > gpurun_out/r02b_select.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02b_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-rope-pass > gpurun_out/r02b_ncu.log 2>&1
tail -3 gpurun_out/r02b_tests.log
