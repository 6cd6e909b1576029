#!/bin/bash
# Fast iteration: GPU parity subset (-k $K) + train bench at several batch sizes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "${K:-fit or forward or collect or aggregate}" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
for b in ${BATCHES:-32 4096 65536}; do
  n=1000000; [ $b -le 64 ] && n=200000
  timeout 300 python bench.py --steps 3 --warmup 2 --batch $b --n $n --no-secondary --no-cpu-baseline > gpurun_out/bench_b$b.log 2>&1
done
eval "${EXTRA:-true}"
tail -2 gpurun_out/pytest_quick.log
for b in ${BATCHES:-32 4096 65536}; do grep -E '^\{' gpurun_out/bench_b$b.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']
    print('B=%6d'%d['config']['global_batch'], 'value=%.3e'%d['value'], 'ms=%.3f'%d['ms_per_step'], 'frac=%.3f'%r['frac'], 'e2e=%.3e'%d['e2e']['value'])
" || tail -3 gpurun_out/bench_b$b.log; done
