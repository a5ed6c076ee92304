cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in 0 1 2; do
  UUV_PDL=$m timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg2_k8 --sizes 4096,16384,65536 > gpurun_out/sweep_pdl$m.jsonl 2>&1; echo "pdl$m exit $?"
done
for m in 0 1 2; do
  UUV_PDL=$m timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_pdl$m.log 2>&1; echo "bench pdl$m exit $?"
done
timeout 300 python scripts/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; cat gpurun_out/e2e_probe.log
