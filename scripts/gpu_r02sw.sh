mkdir -p gpurun_out
python bench.py --config cfg2_sweep --steps 20 --warmup 3 > gpurun_out/r02sw_sweep.jsonl 2> gpurun_out/r02sw_sweep.err
tail -3 gpurun_out/r02sw_sweep.err
cat > /tmp/k3wan.py <<'PY'
import sys; sys.path[:0]=['.']
import torch, bench, paper_2605_20659_b200 as P
dev=torch.device('cuda',0)
base=dict(name="wan", grid=(21,30,52), H=12, d=128, split=(44,42,42), r=64, block=64, sparsity=0.9)
q,k,v,x,params,pe,grid=bench.make_inputs(base,0,12,dev)
st=P.ForwardSettings(P.SparseSettings.for_sparsity(64,grid.size,0.9))
for _ in range(5): P.compensator_branch(x,grid,params,st,pe)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02sw_k3_launches.csv python /tmp/k3wan.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:lowrank_umma_kernel -s 4 -c 1 -o gpurun_out/r02sw_k3 python /tmp/k3wan.py > gpurun_out/r02sw_k3_ncu.log 2>&1
tail -2 gpurun_out/r02sw_k3_ncu.log
