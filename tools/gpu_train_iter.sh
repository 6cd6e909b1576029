#!/bin/bash
# Train-kernel iteration on a B200: fit parity tests (incl. virtual ranks,
# variants, at-size goldens), bench at several batch sizes, phase timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "${K:-fit or peer or variant or c2_ or c3_}" > gpurun_out/pytest_train.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_train.log
for b in ${BATCHES:-4096 8192 65536}; do
  timeout 300 python bench.py --steps 5 --warmup 3 --batch $b --n 1000000 --no-secondary --no-cpu-baseline > gpurun_out/bench_b$b.log 2>&1
done
[ -n "$PHASE" ] && bash tools/phase_timing.sh > gpurun_out/phase_build.log 2>&1 && timeout 300 python tools/phase_timing.py > gpurun_out/phase.log 2>&1
tail -2 gpurun_out/pytest_train.log
for b in ${BATCHES:-4096 8192 65536}; do grep -E '^\{' gpurun_out/bench_b$b.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']
    print('B=%6d'%d['config']['global_batch'], 'value=%.3e'%d['value'], 'kernel_ms=%.4f'%r['kernel_ms_per_step'], 'frac=%.3f'%r['frac'], 'e2e=%.3e'%d['e2e']['value'])
" || tail -3 gpurun_out/bench_b$b.log; done
[ -n "$PHASE" ] && head -60 gpurun_out/phase.log
true
