mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "dit or ulysses or query_block or gate or copy_rows or stage1" > gpurun_out/r02n_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02n_tests.log
timeout 900 python bench.py --config train --steps 10 --warmup 3 > gpurun_out/r02n_train.json 2> gpurun_out/r02n_train.err
timeout 900 python bench.py --config cfg4 --gpus 2 --same-device --backend gloo --steps 2 --warmup 1 > gpurun_out/r02n_cfg4_n2.json 2> gpurun_out/r02n_cfg4_n2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02n_train_launches.csv python bench.py --config train --steps 2 --warmup 1 > /dev/null 2>&1
tail -3 gpurun_out/r02n_tests.log
