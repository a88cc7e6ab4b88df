#!/bin/bash
# A/B timing on one box: tools/ab.sh <libA.so> <libB.so> c1 c5 ...  (alternating runs)
A=$1; B=$2; shift 2
for rep in 1 2; do
  for c in "$@"; do
    echo -n "A "; BISIM_DEV=1 BISIM_LIB=$A bash tools/timing.sh $c
    echo -n "B "; BISIM_DEV=1 BISIM_LIB=$B bash tools/timing.sh $c
  done
done
