mkdir -p gpurun_out
rm -rf gpurun_out/parity
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02as_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02as_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02as_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02as_bench.json 2> gpurun_out/r02as_bench.err
timeout 600 python bench.py --config train --steps 20 --warmup 3 > gpurun_out/r02as_train.json 2> /dev/null
timeout 600 python bench.py --config linear --steps 10 --warmup 3 > gpurun_out/r02as_linear.json 2> /dev/null
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 > gpurun_out/r02as_cfg4.json 2> gpurun_out/r02as_cfg4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02as_ref.json 2> /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:screen|pool_blocks|sparse_attn|lowrank|gate_sum" --csv --log-file gpurun_out/r02as_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
tail -3 gpurun_out/r02as_tests.log
