#!/bin/bash
# ncu evidence for the bench workload (run under gpurun; one GPU).
#   launches_<cfg>.csv       every launch of a short bench run with its device time
#   prof_<cfg>_<kernel>.ncu-rep  --set full capture of one launch of each hot kernel
set -u
OUT=${1:-gpurun_out}
CFG=${CFG:-C1}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_$CFG.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-in-stream --e2e-steps 1 > $OUT/bench_under_ncu.log 2>&1
for k in ${KERNELS:-refresh_tc2 reuse_tc select_heads}; do
  # (reuse_tc: the FIRST launch is kbench's per-head Reuse; its second one runs on the
  # per-KV-group sets, which have far fewer unique rows under GQA)
  skip=1; [ "$k" = reuse_tc ] && skip=0
  ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o $OUT/prof_${CFG}_$k -f \
      python scripts/kbench.py $CFG --iters 2 > $OUT/ncu_$k.log 2>&1
done
if [ "${LMHEAD:-0}" = 1 ]; then
  ncu --set full --clock-control none --import-source on -k regex:lmhead_argmax -s 2 -c 1 -o $OUT/prof_N4_lmhead -f \
      python scripts/bench_lmhead.py --iters 3 > $OUT/ncu_lmhead.log 2>&1
fi
