#!/bin/bash
# dev: A/B the refresh kernel variants built with DLLM_VARIANT (libdllm_<tag>.so)
for f in paper_2512_17077_b200/libdllm.so paper_2512_17077_b200/libdllm_*.so; do
  case $f in *trace*) continue;; esac
  echo "== $f"
  for c in ${CFGS:-C1 C2}; do DLLM_LIB=$f timeout 120 python scripts/kbench.py $c --iters 10 | grep -E "refresh|reuse|select"; done
done
