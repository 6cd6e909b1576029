#!/bin/bash
mkdir -p gpurun_out
for cfg in "20000 32 b32" "1000000 4096 b4096" "1000000 65536 b65536"; do set -- $cfg
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_epoch -s 1 -c 1 -o gpurun_out/prof_train_$3 -f python tools/prof_train.py $1 $2 > gpurun_out/ncu_$3.log 2>&1; echo "$3 rc=$?"; done
