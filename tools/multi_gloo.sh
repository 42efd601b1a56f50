# N>1 logic check on one GPU (gloo: host-side collectives; not a timing)
for mode in "" "--shard triangles" "--shard triangles --merge reduce_scatter"; do
  echo "== mode: $mode"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --backend gloo --no-cpu-baseline --no-hybrid $mode 2>&1 | grep -v Warning | tail -2 | cut -c1-400
done
