cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in new old new old; do
  if [ $v = old ]; then export UUV_B200_LIB=build/variants/lib_task_old.so; else unset UUV_B200_LIB; fi
  timeout 600 python scripts/sweep.py --cases task_cfg4,task_cfg5 --sizes 4096,1048576 >> gpurun_out/sweep_task_$v.jsonl 2>&1; echo "$v exit $?"
done
