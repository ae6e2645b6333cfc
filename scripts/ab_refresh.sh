#!/bin/bash
# dev: alternate Refresh timings of libdllm.so and the DLLM_VARIANT builds given as arguments
# (tags, e.g. DLLM_TC2_SKEW0), CFGS (default "C1 C2"), REPS rounds
for r in $(seq ${REPS:-2}); do
  for c in ${CFGS:-C1 C2}; do
    for t in "" "$@"; do
      f=paper_2512_17077_b200/libdllm${t:+_$t}.so
      DLLM_LIB=$f timeout 120 python scripts/refresh_time.py $c 20
    done
  done
done
