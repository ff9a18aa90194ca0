# Multi-GPU checks for a box with >= 2 GPUs (not available to round 1's gpurun):
# bench.py under torchrun at N = 2, 4, 8 with the fused NVLink paths (default)
# and with the NCCL collectives (SB200_LSA=0); same per-rank workload.
set -x
NG=$(nvidia-smi -L | wc -l)
for N in 2 4 8; do
  [ "$N" -le "$NG" ] || continue
  for LSA in 1 0; do
    SB200_LSA=$LSA timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29600 + N + 10 * LSA)) bench.py --gpus $N --steps 10 --warmup 3 \
      > gpurun_out/scale_${N}_lsa${LSA}.json 2> gpurun_out/scale_${N}_lsa${LSA}.err
    echo "N=$N LSA=$LSA rc=$?"
    tail -c 600 gpurun_out/scale_${N}_lsa${LSA}.json
  done
done
