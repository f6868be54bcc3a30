mkdir -p gpurun_out
rm -rf gpurun_out/parity
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "linear or float32 or select or golden" > gpurun_out/r02f_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02f_tests.log
timeout 600 python bench.py --config linear --steps 10 --warmup 3 > gpurun_out/r02f_linear.json 2> gpurun_out/r02f_linear.err
timeout 300 python scripts/exp_select.py > gpurun_out/r02f_select.log 2>&1
tail -3 gpurun_out/r02f_tests.log
