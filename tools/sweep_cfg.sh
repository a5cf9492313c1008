#!/bin/bash
# A/B the compiled-in sort / unique variants on C2 (one line per config).
out=${1:-gpurun_out/sweep.txt}
: > $out
for s in ${SORTS:-A B C D E F G H I}; do
  r=$(RMX_SORT_CFG=$s timeout 120 python tools/profile_step.py --config C2 --steps 3 2>&1 | awk '/sort_pass/ && $2>0.05 {n++; t+=$2} /unique/ {u=$2} /total/ {tot=$2} /build_rows/ {b=$2} END {printf "passes=%d pass_avg=%.3f unique=%.3f build=%.3f total=%.3f", n, t/n, u, b, tot}')
  echo "sort=$s $r" >> $out
done
for u in ${UNIQS:-A B C D}; do
  r=$(RMX_UNIQ_CFG=$u timeout 120 python tools/profile_step.py --config C2 --steps 3 2>&1 | awk '/sort_pass/ && $2>0.05 {n++; t+=$2} /unique/ {u=$2} /total/ {tot=$2} END {printf "pass_avg=%.3f unique=%.3f total=%.3f", t/n, u, tot}')
  echo "uniq=$u $r" >> $out
done
cat $out
