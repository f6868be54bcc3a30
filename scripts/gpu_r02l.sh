mkdir -p gpurun_out
timeout 600 python bench.py --config skew --steps 6 --warmup 2 > gpurun_out/r02l_skew.jsonl 2> gpurun_out/r02l_skew.err
timeout 900 ncu --set full --clock-control none -k 'regex:sparse_attn_fixed' -c 1 -o gpurun_out/r02l_k2_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-rope-pass > gpurun_out/r02l_k2_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k 'regex:sparse_attn_fixed' -c 1 -o gpurun_out/r02l_k2_cfg1_full -f python bench.py --config cfg1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-rope-pass > gpurun_out/r02l_k2_cfg1_full.log 2>&1
tail -2 gpurun_out/r02l_k2_full.log
