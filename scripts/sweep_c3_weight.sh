#!/bin/bash
# dev: C3 mixed-launch SM split sweep (DLLM_MIXED_REFRESH_WEIGHT scales the Refresh phase estimate)
for r in 1 2; do for w in ${WEIGHTS:-0.8 0.9 1.0 1.1 1.25}; do
  DLLM_MIXED_REFRESH_WEIGHT=$w python bench.py --config C3 --no-configs --no-cpu-baseline --e2e-steps 1 --steps 10 --warmup 3 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']['mixed']; print('weight $w', 'C3 step', round(d['ms_per_step']*1000,1), 'us; mixed', round(k['us'],1), 'us frac', round(k['frac'],3))"
done; done
