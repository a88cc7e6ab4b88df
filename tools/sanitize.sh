#!/bin/bash
# compute-sanitizer passes over tools/sanitize_cases.py; logs under the
# directory given as $1 (default gpurun_out/).  Each tool's summary line
# ("ERROR SUMMARY: N errors") is what profiles/ records.
out=${1:-gpurun_out}
mkdir -p "$out"
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 \
    python tools/sanitize_cases.py > "$out/sanitize_$tool.log" 2>&1
  echo "$tool rc=$? $(grep -h 'ERROR SUMMARY\|SANITIZE_CASES_OK' "$out/sanitize_$tool.log" | tr '\n' ' ')"
done
