#!/bin/bash
# One ncu --set full capture of a kernel (regex) launched by a command;
# writes <out>.ncu-rep plus raw / source / details CSVs under gpurun_out/.
#   bash scripts/ncu_top.sh <out-name> <kernel-regex> <launch-skip> <command...>
OUT="$1"; K="$2"; SKIP="$3"; shift 3
ncu --set full --clock-control none --import-source on -k "regex:$K" --launch-skip "$SKIP" \
    --launch-count 1 -o "gpurun_out/$OUT" "$@" > "gpurun_out/$OUT.log" 2>&1
for page in raw source details; do
  ncu -i "gpurun_out/$OUT.ncu-rep" --page $page --csv > "gpurun_out/${OUT}_$page.csv" 2>&1
done
