#!/bin/bash
# compute-sanitizer over every kernel family (profiles/sanitize.py), one tool x
# section per process; logs + a one-line summary per run into $OUT.
OUT=${OUT:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for what in query train render dist; do
    log="$OUT/${tool}_${what}.log"
    timeout 900 $CS --tool $tool --print-limit 20 python profiles/sanitize.py $what > "$log" 2>&1
    rc=$?
    echo "$tool $what rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$log" | tr '\n' ' ')" | tee -a "$OUT/summary.txt"
  done
done
