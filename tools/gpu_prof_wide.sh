#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wide_launches.csv python tools/prof_wide.py 65536 > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 30 -c 5 -o gpurun_out/prof_wide_gemm -f python tools/prof_wide.py 65536 > /dev/null 2>&1; echo rc=$?
