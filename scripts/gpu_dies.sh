for v in default _ab/dies1.so _ab/dies2.so default _ab/dies1.so _ab/dies2.so; do
  if [ $v = default ]; then python scripts/exp_k2_order.py; else ROPESLR_LIBRARY=$v python scripts/exp_k2_order.py; fi
done
for v in default _ab/dies1.so _ab/dies2.so; do
  if [ $v = default ]; then unset ROPESLR_LIBRARY; else export ROPESLR_LIBRARY=$v; fi
  N=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:sparse_attn_fixed -s 3 -c 1 --csv python scripts/exp_k2_order.py 2>/dev/null | grep -E "dram__bytes|gpu__time|lts__" | awk -F'","' '{print "'$v'", $(NF-2), $NF}'
done
