#!/bin/bash
# Process-level A/B of two library builds (fresh device allocations every run,
# which matters: latency-bound configs move by several % with buffer placement).
#   tools/ab_proc.sh ab/libA.so ab/libB.so REPS c3 c1 ...
# prints one "config lib alg_ms" line per run; summarise with tools/ab_summary.py
A=$1; B=$2; R=$3; shift 3
for c in "$@"; do
  for rep in $(seq 1 $R); do
    if [ $((rep % 2)) -eq 1 ]; then order="A B"; else order="B A"; fi
    for L in $order; do
      if [ $L = A ]; then lib=$A; else lib=$B; fi
      BISIM_DEV=1 BISIM_LIB=$lib timeout 600 python tools/run_config.py $c sparse 2 2>/dev/null | tail -1 | \
        sed -n "s/.*alg=\([0-9.]*\)ms.*/$c $L \1/p"
    done
  done
done
