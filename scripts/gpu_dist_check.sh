# Multi-rank bench path on ONE GPU: 2 and 3 ranks over gloo (host-staged exchanges)
set -x
for N in 2 3; do
SB200_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
  --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps 3 --warmup 3 \
  --dofs 2e7 --mesh-k 30 > gpurun_out/dist_check_$N.json 2> gpurun_out/dist_check_$N.err; echo "world $N rc=$?"
tail -c 1500 gpurun_out/dist_check_$N.json
done
