#!/bin/bash
# preprocessing / loop timing of several library builds on one box:
#   tools/pre_ab.sh CONFIG REPS ab/libX.so ab/libY.so ...
c=$1; R=$2; shift 2
for r in $(seq 1 $R); do for L in "$@"; do echo "$L $(BISIM_LIB=$L tools/timing.sh $c)"; done; done
