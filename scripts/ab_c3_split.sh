#!/bin/bash
# dev: C3 mixed-launch SM split sweep (DLLM_MIXED_REFRESH_WEIGHT scales the Refresh share)
for w in 0.9 1.0 1.1; do
  echo "== weight $w"
  DLLM_MIXED_REFRESH_WEIGHT=$w timeout 300 python bench.py --config C3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels']['mixed']['us'])"
done
