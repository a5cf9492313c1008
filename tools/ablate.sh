#!/bin/bash
# Sort-pass ablations on C2 (timings only; results invalid when RMX_ABLATE != 0).
for cfg in ${SORTS:-I}; do for ab in 0 1 2 4 3 5 6 7; do
  r=$(RMX_SORT_CFG=$cfg RMX_ABLATE=$ab timeout 120 python tools/profile_step.py --config C2 --steps 3 2>&1 | awk '/sort_pass/ && $2>0.05 {n++; t+=$2} END {printf "passes=%d pass_avg=%.3f", n, t/n}')
  echo "sort=$cfg ablate=$ab $r"
done; done
