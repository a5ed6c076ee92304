cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/bench_cem.py --envs 512,65536,1048576 --iterations 5 > gpurun_out/bench_cem.jsonl 2> gpurun_out/bench_cem.err
echo "bench_cem exit $?"; cat gpurun_out/bench_cem.jsonl; tail -3 gpurun_out/bench_cem.err
