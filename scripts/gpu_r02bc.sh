mkdir -p gpurun_out
rm -rf gpurun_out/parity
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02bc_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02bc_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02bc_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02bc_bench.json 2> gpurun_out/r02bc_bench.err
timeout 600 python bench.py --config linear --steps 10 --warmup 3 > gpurun_out/r02bc_linear.json 2> /dev/null
timeout 600 python bench.py --config train --steps 20 --warmup 3 > gpurun_out/r02bc_train.json 2> /dev/null
tail -3 gpurun_out/r02bc_tests.log
