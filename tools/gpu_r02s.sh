#!/bin/bash
O=gpurun_out; mkdir -p $O
echo default > $O/r02s_padd.txt; timeout 300 python tools/exp/padd_forms.py fused,fused2 18,20,22 >> $O/r02s_padd.txt 2>&1
for v in f128_5 f128_6 f256_2 f256_3 f64_8; do
  echo $v >> $O/r02s_padd.txt
  GECC_LIB=$PWD/paper_2501_03245_b200/lib/libgecc_b200_$v.so timeout 300 python tools/exp/padd_forms.py fused,fused2 18,20,22 >> $O/r02s_padd.txt 2>&1
done
cat $O/r02s_padd.txt
