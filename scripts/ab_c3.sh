#!/bin/bash
# dev: C3 mixed-step time for libdllm.so and the given tags
for r in 1 2; do for t in "" "$@"; do
  DLLM_LIB=paper_2512_17077_b200/libdllm${t:+_$t}.so python bench.py --config C3 --no-configs --no-cpu-baseline --e2e-steps 1 --steps 10 --warmup 3 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']['mixed']; print('${t:-libdllm}', 'C3 step', round(d['ms_per_step']*1000,1), 'us; mixed', round(k['us'],1), 'us frac', round(k['frac'],3))"
done; done
