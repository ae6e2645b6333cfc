#!/bin/bash
# dev: A/B of the Reuse dynamic scheduler (kbench C1/C2/C4, bench C3 with SM-split weights)
timeout 700 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py tests/test_gpu_fused_select.py -x -q > gpurun_out/pytest_rdyn.log 2>&1
CFGS="C1 C2 C4" bash scripts/ab_variants.sh > gpurun_out/ab_rdyn.log 2>&1
for L in paper_2512_17077_b200/libdllm.so paper_2512_17077_b200/libdllm_DLLM_RTC_DYNSCHED0.so; do
  for w in 1.0 0.8 1.25; do
    echo "== $L weight $w" >> gpurun_out/c3_split.log
    DLLM_LIB=$L DLLM_MIXED_REFRESH_WEIGHT=$w timeout 300 python bench.py --config C3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels']['mixed']['us'])" >> gpurun_out/c3_split.log 2>&1
  done
done
DLLM_LIB=paper_2512_17077_b200/libdllm.so timeout 300 python bench.py --config C3 --no-mixed --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 > gpurun_out/c3_nomixed.json
