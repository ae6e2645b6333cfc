for r in 1 2; do for t in "" prev; do
  DLLM_LIB=paper_2512_17077_b200/libdllm${t:+_$t}.so python bench.py --no-configs --no-cpu-baseline --e2e-steps 1 --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('${t:-new}', round(d['ms_per_step']*1000,1), 'us/step', round(d['value']), 'req/s', 'refresh', round(d['kernels']['refresh']['us'],1))"
done; done
