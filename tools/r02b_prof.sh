#!/bin/bash
# full ncu capture of k_cycle for two builds (tags old / new)
for v in old new; do
  L=$PWD/paper_2304_13541_b200/libdstack_$v.so; [ $v = new ] && L=$PWD/paper_2304_13541_b200/libdstack.so
  DSTACK_LIB=$L bash tools/prof_k.sh k_cycle kc_$v
done
ls -la gpurun_out/
exit 0
