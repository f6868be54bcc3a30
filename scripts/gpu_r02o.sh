mkdir -p gpurun_out
rm -rf gpurun_out/parity
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02o_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02o_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02o_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err
timeout 600 python bench.py --config train --steps 20 --warmup 3 > gpurun_out/r02o_train.json 2> gpurun_out/r02o_train.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02o_train_launches.csv python bench.py --config train --steps 2 --warmup 1 > /dev/null 2>&1
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 > gpurun_out/r02o_cfg4.json 2> gpurun_out/r02o_cfg4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02o_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
tail -3 gpurun_out/r02o_tests.log
