mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "dit or ulysses or query_block or gate or copy_rows" > gpurun_out/r02m_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02m_tests.log
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 > gpurun_out/r02m_cfg4.json 2> gpurun_out/r02m_cfg4.err
timeout 900 python bench.py --config cfg4 --gpus 2 --same-device --backend gloo --steps 2 --warmup 1 > gpurun_out/r02m_cfg4_n2.json 2> gpurun_out/r02m_cfg4_n2.err
tail -3 gpurun_out/r02m_tests.log
