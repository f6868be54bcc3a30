mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compensator.py tests/test_gpu_parity.py tests/test_gpu_host.py -x -q 2>&1 | tail -4
python bench.py --config cfg2_sweep --steps 20 --warmup 3 > gpurun_out/r02k3_sweep.jsonl 2> gpurun_out/r02k3_sweep.err
tail -2 gpurun_out/r02k3_sweep.err
cat > /tmp/k3wan.py <<'PY'
import sys; sys.path[:0]=['.']
import torch, bench, paper_2605_20659_b200 as P
dev=torch.device('cuda',0)
for base in (dict(name="wan", grid=(21,30,52), H=12, d=128, split=(44,42,42), r=64, block=64, sparsity=0.9),
             dict(name="c3", grid=(33,45,80), H=24, d=128, split=(16,56,56), r=64, block=128, sparsity=0.9)):
    q,k,v,x,params,pe,grid=bench.make_inputs(base,0,base["H"],dev)
    st=P.ForwardSettings(P.SparseSettings.for_sparsity(base["block"],grid.size,0.9))
    for _ in range(5): P.compensator_branch(x,grid,params,st,pe)
    torch.cuda.synchronize()
    del q,k,v
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02k3_launches.csv python /tmp/k3wan.py > /dev/null 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02k3_bench.json 2> gpurun_out/r02k3_bench.err; tail -2 gpurun_out/r02k3_bench.err
