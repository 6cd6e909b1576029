#!/bin/bash
# ncu launch list + full captures of the top kernels (one GPU, short commands).
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_epoch -s 1 -c 1 \
    -o gpurun_out/prof_train -f $B --no-secondary > gpurun_out/ncu_train.log 2>&1
echo "train capture rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd_fast|aggregate_kernel|fwd_exact" -s 3 -c 3 \
    -o gpurun_out/prof_infer -f $B > gpurun_out/ncu_infer.log 2>&1
echo "infer capture rc=$?"
ls -la gpurun_out
