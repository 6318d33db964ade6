for v in r1 ef1d91f a63ce68 aff2c45 8355da6 new; do
  L=$PWD/paper_2304_13541_b200/libdstack_$v.so; [ $v = new ] && L=$PWD/paper_2304_13541_b200/libdstack.so
  DSTACK_LIB=$L python tools/dbg_hook.py $v 2>&1 | tail -2
done
