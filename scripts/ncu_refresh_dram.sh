#!/bin/bash
# dev: DRAM bytes + duration of one Refresh launch (ncu) for libdllm.so and the given build tags
for t in "" "$@"; do
  for c in ${CFGS:-C1 C2}; do
    DLLM_LIB=paper_2512_17077_b200/libdllm${t:+_$t}.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:refresh_tc2 -s 2 -c 1 --csv python scripts/refresh_time.py $c 3 2>/dev/null |
      grep -E "dram__|gpu__time" | awk -F'","' -v t="${t:-libdllm}" -v c=$c '{print t, c, $(NF-2), $NF}'
  done
done
