mkdir -p gpurun_out
for i in 1 2 3; do timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02ab_bench$i.json 2> gpurun_out/r02ab_bench$i.err; done
ROPESLR_SCREEN=0 timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02ab_bench_noscreen.json 2> /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:ropeslr|tc::|lu::|screen|pool" --csv --log-file gpurun_out/r02ab_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
