mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:linear_state|linear_apply' -c 2 -o gpurun_out/r02i_linear_full -f python bench.py --config linear --steps 1 --warmup 1 > gpurun_out/r02i_linear_full.log 2>&1
tail -2 gpurun_out/r02i_linear_full.log
