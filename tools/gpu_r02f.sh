#!/bin/bash
# r02: the full bench line (default args), then compute-sanitizer over every kernel family.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02f
mkdir -p $O
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
tail -c 1500 $O/bench.json; tail -3 $O/bench.err
bash tools/sanitize.sh
