# the multi-rank bench path (torchrun, 2 ranks) on ONE GPU with the gloo backend: exercises the sharding, the
# per-step all-reduce, max-over-ranks timing and every leg's multi-rank code (numbers are not scaling results)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
BENCH_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_2r.json 2> gpurun_out/bench_2r.err
echo "rc=$?"; tail -c 600 gpurun_out/bench_2r.json; grep -v "^\s*$" gpurun_out/bench_2r.err | tail -5
