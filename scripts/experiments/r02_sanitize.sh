#!/bin/bash
# Round 2: compute-sanitizer memcheck / racecheck / synccheck over every kernel incl. the round-2 paths.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout -s KILL 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/san_$tool.log 2>&1
  echo rc=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize.*ok|Error|error" gpurun_out/san_$tool.log | head -8
done
