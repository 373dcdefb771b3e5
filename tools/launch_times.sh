#!/bin/bash
# usage: tools/launch_times.sh <command...>  — per-launch kernel durations (ncu, cold, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none --csv "$@" 2>/dev/null \
  | awk -F'","' 'NR>1 && $13=="gpu__time_duration.sum" {gsub(/"/,"",$15); k=$5; sub(/\(.*/,"",k); printf "%-60s %12.1f us\n", k, $15/1000}'
