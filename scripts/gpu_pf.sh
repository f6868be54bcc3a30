for v in default _ab/pf2.so _ab/pf4.so _ab/pf8.so default _ab/pf4.so; do
  if [ $v = default ]; then unset ROPESLR_LIBRARY; else export ROPESLR_LIBRARY=$v; fi
  python scripts/exp_k2_order.py
done
for v in default _ab/pf4.so _ab/pf8.so; do
  if [ $v = default ]; then unset ROPESLR_LIBRARY; else export ROPESLR_LIBRARY=$v; fi
  N=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:sparse_attn_fixed -s 3 -c 1 --csv python scripts/exp_k2_order.py 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' '{print "'$v'", $(NF-2), $NF}'
done
