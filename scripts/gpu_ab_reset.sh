cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_ab.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_ab.log
for rep in 1 2; do for v in new old; do
  if [ $v = new ]; then unset UUV_B200_LIB; else export UUV_B200_LIB=build/variants/lib_old.so; fi
  echo "== $v"; timeout 300 python scripts/probes/reset_cost.py 2>&1 | tail -4
  timeout 300 python scripts/bench_cem.py --envs 512 --iterations 5 --cpu-steps 2 2>&1 | head -1 | cut -c1-200
done; done
unset UUV_B200_LIB
AB_OLD=old bash scripts/gpu_task_ab.sh
