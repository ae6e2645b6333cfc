#!/bin/bash
# dev: Reuse per-launch time in a stream of 31 (bench.py's in-stream figure) for libdllm.so and the given tags
for r in 1 2; do for c in ${CFGS:-C1 C2}; do for t in "" "$@"; do
  DLLM_LIB=paper_2512_17077_b200/libdllm${t:+_$t}.so python bench.py --config $c --no-configs --no-cpu-baseline --e2e-steps 1 --steps 5 --warmup 3 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']['reuse']; print('${t:-libdllm}', '$c', 'reuse single', round(k['us'],1), 'in-stream', round(k['us_in_stream'],1))"
done; done; done
