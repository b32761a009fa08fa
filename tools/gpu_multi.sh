# tools/gpu_multi.sh — the first session on a box with >= 2 GPUs (none has been available so far):
# the data-parallel path end to end. Writes gpurun_out/multi_*.log.
#   bash tools/gpu_multi.sh [N]      (N GPUs, default: all visible)
N=${1:-$(nvidia-smi -L | wc -l)}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/multi_build.log 2>&1
# 1. replicas vs the oracle's replica protocol at W = 2 (C13, C14, C15, and the C17 device kernel)
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -s > gpurun_out/multi_dist.log 2>&1
echo "dist rc $?" >> gpurun_out/multi_dist.log
# 2. scaling (the bench line's run.sync_path says whether NCCL gave the C17 kernel a multicast
#    team: 3 = NVLS multimem, 2 = NVLink loads/stores): the paper's protocol (C13) via NCCL, via the C17 kernel, and C15 overlapped
for n in 2 4 8; do
  [ "$n" -gt "$N" ] && continue
  for variant in "" "--sync-device 1" "--sync-overlap 1" "--sync-overlap 1 --sync-device 1"; do
    tag=$(echo "n${n} ${variant}" | tr ' -' '__')
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
        --master-port $((29600 + n)) bench.py --gpus "$n" --steps 5 --warmup 3 $variant \
        > "gpurun_out/multi_bench_${tag}.log" 2>&1
    echo "rc $?" >> "gpurun_out/multi_bench_${tag}.log"
  done
done
