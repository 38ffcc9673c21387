#!/bin/bash
# A/B of training-step kernels across library builds (NASG_LIB), ncu launch times of
# one config-3 step: usage profiles/ab_ncu_train.sh lib_exp/old lib_exp/new ...
for v in "$@"; do
  for i in 1 2; do
    NASG_LIB=$PWD/paper_2303_08064_b200/$v/libnasg_b200.so AB_T=262144 python profiles/ab_train.py $v | cut -c1-140
  done
  NASG_LIB=$PWD/paper_2303_08064_b200/$v/libnasg_b200.so ncu --metrics gpu__time_duration.sum --clock-control none \
     -k regex:"classify|train_tc|adam" -s 5 -c 5 python profiles/capture_train3.py 2>&1 | grep -E "^  [a-z_A-Z]|duration" | \
     paste - - | awk -v v=$v '{print v, $1, $(NF)}'
done
