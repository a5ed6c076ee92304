# Exercise bench.py's multi-rank path on a single-GPU box: 2 ranks share GPU 0 over gloo.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
UUV_BENCH_GPU_OVERRIDE=0 UUV_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 200 --warmup 5 > gpurun_out/bench_2rank.log 2>&1
echo "2-rank exit $?"; tail -2 gpurun_out/bench_2rank.log | cut -c1-400
UUV_BENCH_GPU_OVERRIDE=0 UUV_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_2rank_ref.log 2>&1
echo "2-rank ref exit $?"; tail -2 gpurun_out/bench_2rank_ref.log | cut -c1-300
