mkdir -p gpurun_out
rm -rf gpurun_out/parity
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02k_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02k_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err
timeout 600 python bench.py --config linear --steps 10 --warmup 3 > gpurun_out/r02k_linear.json 2> gpurun_out/r02k_linear.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:linear|gate" --csv --log-file gpurun_out/r02k_linear_launches.csv python bench.py --config linear --steps 2 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:linear_apply|linear_state' -c 2 -o gpurun_out/r02k_linear_full -f python bench.py --config linear --steps 1 --warmup 1 > gpurun_out/r02k_linear_full.log 2>&1
tail -3 gpurun_out/r02k_tests.log
