# Interleaved A/B of the task-step kernels (+ CEM) between the in-tree build and
# build/variants/lib_$AB_OLD.so on one box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.jsonl
for rep in 1 2; do for v in new ${AB_OLD:-old}; do
  if [ $v = new ]; then unset UUV_B200_LIB; else export UUV_B200_LIB=build/variants/lib_$v.so; fi
  timeout 600 python scripts/sweep.py --cases task_cfg4,task_cfg5 --sizes 4096,65536,1048576 >> gpurun_out/ab_$v.jsonl 2>&1; echo "$v exit $?"
done; done
