#!/bin/bash
# usage: tools/timing.sh c1 c5 ...   (one bench line per config, summarised)
for c in "$@"; do
  BISIM_DEV=1 timeout 600 python bench.py --config $c --steps 2 --warmup 1 --no-cpu 2>&1 | tail -1 | python -c "
import json,sys
t=sys.stdin.read()
try:
    d=json.loads(t)
except Exception:
    print('$c', 'FAILED', t[-300:]); sys.exit()
print('$c', 'ms=%.2f R=%d us/round=%.2f pre=%.2f label=%.2f alg=%.2f GB/s=%.1f ok=%s' % (d['ms_per_step'], d['config']['supersteps'], d['per_round_us'], d['phase_ms']['pre'], d['phase_ms']['label'], d['phase_ms']['alg'], d['roofline']['achieved'], d.get('parity')))"
done
