#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every product
# kernel (tools/sanitize_cases.py); logs to gpurun_out/, summaries copied to
# profiles/ by hand.
out=${1:-gpurun_out}
mkdir -p "$out"
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_cases.py > "$out/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$out/sanitize_$tool.log"
  tail -4 "$out/sanitize_$tool.log"
done
