#!/bin/bash
# dev: A/B the refresh implementations selectable at run time
for impl in ${IMPLS:-tc2 tc1}; do
  echo "== refresh impl $impl"
  for c in ${CFGS:-C1 C2}; do DLLM_REFRESH_IMPL=$impl timeout 120 python scripts/kbench.py $c --iters 10 | grep refresh; done
done
