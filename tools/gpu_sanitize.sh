#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py (1 GPU).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
timeout 300 python tools/sanitize.py > gpurun_out/sanitizer/plain.txt 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/sanitizer/plain.txt
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py > gpurun_out/sanitizer/$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|complete" gpurun_out/sanitizer/$tool.txt | tail -3
done
