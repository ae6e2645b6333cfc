for r in 1 2; do for t in "" prev; do
  DLLM_LIB=paper_2512_17077_b200/libdllm${t:+_$t}.so python scripts/kbench.py C2 --iters 20 2>/dev/null | grep -E "reuse_group_sets|reuse  :" | sed "s/^/${t:-new} /"
done; done
