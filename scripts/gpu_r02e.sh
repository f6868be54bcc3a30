mkdir -p gpurun_out
rm -rf gpurun_out/parity
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02e_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02e_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
timeout 300 python scripts/exp_select.py > gpurun_out/r02e_select.log 2>&1
tail -3 gpurun_out/r02e_tests.log
