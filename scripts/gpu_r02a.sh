set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02a_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02a_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
timeout 600 python bench.py --gpus 2 --same-device --backend gloo --steps 5 --warmup 3 --no-e2e --no-rope-pass --no-cpu-baseline > gpurun_out/r02a_bench_n2.json 2> gpurun_out/r02a_bench_n2.err
tail -3 gpurun_out/r02a_tests.log
