mkdir -p gpurun_out
rm -rf gpurun_out/parity
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02f_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02f_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
timeout 600 python bench.py --config train --steps 20 --warmup 3 > gpurun_out/r02f_train.json 2> /dev/null
timeout 600 python bench.py --config linear --steps 10 --warmup 3 > gpurun_out/r02f_linear.json 2> /dev/null
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 > gpurun_out/r02f_cfg4.json 2> gpurun_out/r02f_cfg4.err
timeout 900 python bench.py --config cfg2_sweep --steps 20 --warmup 3 > gpurun_out/r02f_sweep.jsonl 2> /dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02f_ref.json 2> /dev/null
timeout 900 python bench.py --gpus 2 --same-device --backend gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_n2.json 2> gpurun_out/r02f_n2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:screen|pool_blocks|sparse_attn|lowrank|gate_sum" --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/r02f_tests.log
cat gpurun_out/r02f_smoke.log | tail -1
