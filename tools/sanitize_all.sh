#!/bin/bash
# usage: tools/sanitize_all.sh <racecheck|synccheck|memcheck>  (one tool per gpurun call)
tool=$1
out=gpurun_out/sanitize_$tool.log
: > $out
for r in resident grid dense chain fused ws; do
  env="ODX_GRID_RESIDENT=1"
  [ $r = chain ] && env="ODX_GRID_RESIDENT=0"
  [ $r = fused ] && env="ODX_GRID_RESIDENT=0 ODX_CHAIN=0"
  [ $r = ws ] && env="ODX_GRID_RESIDENT=0 ODX_CHAIN=0 ODX_FUSED_TILED=0"
  echo "=== $tool $r ($env)" >> $out
  env $env timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $r >> $out 2>&1
  echo "rc=$?" >> $out
done
