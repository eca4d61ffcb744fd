#!/bin/bash
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/san_$tool.log 2>&1
  echo rc=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize run ok|Error|error" gpurun_out/san_$tool.log | head -8
done
