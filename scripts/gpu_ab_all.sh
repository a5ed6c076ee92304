# A/B of the in-tree build vs build/variants/lib_old.so: physics sweep + task sweep, interleaved.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.jsonl
for rep in 1 2; do for v in new old; do
  if [ $v = new ]; then unset UUV_B200_LIB; else export UUV_B200_LIB=build/variants/lib_old.so; fi
  timeout 600 python scripts/sweep.py --cases ${AB_CASES:-cfg2,bluerov,cfg5_physics,cfg2_k8,cfg3} --sizes ${AB_SIZES:-4096,1048576} >> gpurun_out/ab_$v.jsonl 2>&1
  timeout 600 python scripts/sweep.py --cases task_cfg4,task_cfg5 --sizes ${AB_SIZES:-4096,1048576} >> gpurun_out/ab_$v.jsonl 2>&1
  echo "$v exit $?"
done; done
