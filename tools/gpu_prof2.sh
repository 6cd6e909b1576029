#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_epoch -s 1 -c 1 -o gpurun_out/prof_train_b32 -f python tools/prof_train.py 20000 32 > gpurun_out/ncu1.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_epoch -s 1 -c 1 -o gpurun_out/prof_train_b4096 -f python tools/prof_train.py 1000000 4096 > gpurun_out/ncu2.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:shuffle -s 1 -c 1 -o gpurun_out/prof_shuffle -f python tools/prof_train.py 1000000 65536 > gpurun_out/ncu3.log 2>&1; echo rc=$?
