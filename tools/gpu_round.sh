#!/bin/bash
# Round evidence: full GPU tests, smoke, default bench, ncu launch list + full
# captures of the top kernels. Everything lands in gpurun_out/.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv $B --no-secondary > gpurun_out/ncu_launch_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_epoch -s 1 -c 1 -o gpurun_out/prof_train -f $B --no-secondary > gpurun_out/ncu_train.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_fast|aggregate_kernel|w16_gemm|w16_update|qt_fold|qt_snapshot" -s 1 -c 10 -o gpurun_out/prof_other -f $B > gpurun_out/ncu_other.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -c 600 gpurun_out/bench.log
