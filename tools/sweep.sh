#!/bin/bash
# usage: sweep.sh "ENV1" "ENV2" ... -- configs
envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
for rep in 1 2; do for c in "$@"; do for e in "${envs[@]}"; do
  echo -n "[$e] "; env $e bash tools/timing.sh $c
done; done; done
