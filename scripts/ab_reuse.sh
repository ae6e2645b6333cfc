#!/bin/bash
# dev: alternate Reuse timings of libdllm.so and the builds given as tags (libdllm_<tag>.so)
for r in $(seq ${REPS:-2}); do
  for c in ${CFGS:-C1 C2 C4}; do
    for t in "" "$@"; do
      DLLM_LIB=paper_2512_17077_b200/libdllm${t:+_$t}.so timeout 180 python scripts/reuse_time.py $c 30
    done
  done
done
