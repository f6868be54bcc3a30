set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_dit.py -x -q 2>&1 | tail -5
python bench.py --config cfg4 --steps 3 --warmup 3 > gpurun_out/r02ln_cfg4.json 2> gpurun_out/r02ln_cfg4.err; tail -2 gpurun_out/r02ln_cfg4.err
cat gpurun_out/r02ln_cfg4.json
python scripts/exp_dit_profile.py 2>&1 | head -25 > gpurun_out/r02ln_dit_profile.txt
