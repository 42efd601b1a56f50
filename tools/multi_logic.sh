#!/bin/bash
# N>1 host-logic check of bench.py on ONE GPU (gloo process group, virtual-rank handles; not a measurement):
# sensor shards (default), triangle shards (all-reduce / reduce-scatter readback ranges), mixed partition.
set -e
port=29541
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
  --master-port $((port++)) bench.py --gpus $n --steps 4 --warmup 3 --logic-check --no-cpu-baseline "$@" 2>&1 | grep '^{' | cut -c1-300; }
run 2
run 2 --shard triangles
run 2 --shard triangles --merge reduce_scatter
run 4 --shard mixed --emitter-groups 2
