#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_driver.py); the summaries land in
# gpurun_out/sanitize/ (one log per tool x case, the last lines kept).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/sanitize
mkdir -p $O
for c in fused hybrid resident cg stream c5; do
  python tools/sanitize_driver.py $c > $O/plain_$c.txt 2>&1 || { echo "plain $c failed"; continue; }
  for t in memcheck racecheck synccheck; do
    timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_driver.py $c > $O/${t}_$c.log 2>&1
    echo "$t $c rc $? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $O/${t}_$c.log | tail -2 | tr '\n' ' ')"
    tail -c 3000 $O/${t}_$c.log > $O/${t}_$c.tail; rm -f $O/${t}_$c.log
  done
done
