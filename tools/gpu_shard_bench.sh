#!/bin/bash
# the sharded bench path (torchrun, 2-3 ranks) on ONE GPU: collectives through the library's host
# transport over gloo (NCCL refuses two ranks on one device)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/shard
mkdir -p $O
for spec in "2 128" "3 128" "2 256"; do
  set -- $spec
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29500 + $1 + $2)) \
    bench.py --gpus $1 --steps 2 --warmup 3 --size $2 --transport host --no-c5 --no-sweep --no-cpu-baseline \
    > $O/shard_$1_$2.json 2> $O/shard_$1_$2.err
  echo "ranks $1 size $2 rc $?"
  python -c "
import json,sys
d=json.loads(open('$O/shard_$1_$2.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','n_gpus','scaling','iterations_per_step','converged','true_resid_over_eps')}, d['config']['parallelism'])
" 2>&1 | tail -2
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29650 \
  bench.py --gpus 2 --steps 2 --warmup 3 --size 128 --transport host --replicas --no-c5 --no-sweep --no-cpu-baseline \
  > $O/rep_2_128.json 2> $O/rep_2_128.err; echo "replicas rc $?"; tail -c 600 $O/rep_2_128.json
timeout 600 python bench.py --steps 2 --warmup 3 --size 128 --no-c5 --no-sweep --no-cpu-baseline > $O/single_128.json 2>&1
python -c "
import json
d=json.loads(open('$O/single_128.json').read().strip().splitlines()[-1])
print('single', {k: d[k] for k in ('value','ms_per_step','iterations_per_step','true_resid_over_eps')})
"
for f in $O/*.err; do tail -n 3 $f; done
