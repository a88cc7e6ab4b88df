#!/bin/bash
# Process-level A/B of two developer-knob settings of the same library:
#   tools/ab_env.sh "BISIM_BATCH_C=8192" "BISIM_BATCH_C=4096" REPS c5 c4l ...
# output format as tools/ab_proc.sh (summarise with tools/ab_summary.py)
EA=$1; EB=$2; R=$3; shift 3
for c in "$@"; do
  for rep in $(seq 1 $R); do
    if [ $((rep % 2)) -eq 1 ]; then order="A B"; else order="B A"; fi
    for L in $order; do
      if [ $L = A ]; then e=$EA; else e=$EB; fi
      env BISIM_DEV=1 $e timeout 600 python tools/run_config.py $c sparse 2 2>/dev/null | tail -1 | \
        sed -n "s/.*alg=\([0-9.]*\)ms.*/$c $L \1/p"
    done
  done
done
