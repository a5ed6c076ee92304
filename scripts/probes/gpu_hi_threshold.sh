cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.jsonl
for rep in 1 2; do for v in hi lo; do
  if [ $v = hi ]; then export UUV_HI_OCC_MIN_ENVS=0; else export UUV_HI_OCC_MIN_ENVS=999999999; fi
  timeout 600 python scripts/sweep.py --cases cfg2,cfg5_physics,cfg2_k8 --sizes 16384,65536,131072,262144,1048576 >> gpurun_out/ab_$v.jsonl 2>&1
done; done
