# functional run of the bench's N>1 path on one GPU: 2 torchrun ranks on the same device (BENCH_SHARE_DEVICE=1,
# gloo timing collectives, the CUDA IPC peer-store exchange); one JSON line from rank 0
set -x
BENCH_SHARE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --quick --no-cpu-baseline \
  > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err; echo "bench n2 rc=$?"
tail -c 600 gpurun_out/bench_n2_shared.json; grep -i "fall\|error\|Traceback" gpurun_out/bench_n2_shared.err | head
