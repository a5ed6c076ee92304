# Interleaved A/B of library builds on one box.  AB_VARIANTS: names under
# build/variants/lib_<name>.so, plus "new" for the in-tree build.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.jsonl
CASES=${AB_CASES:-cfg2,bluerov,cfg5_physics,cfg2_k8,cfg3}
SIZES=${AB_SIZES:-4096,1048576,4194304}
for rep in 1 2; do
  for v in ${AB_VARIANTS:-new old}; do
    if [ $v = new ]; then unset UUV_B200_LIB; else export UUV_B200_LIB=build/variants/lib_$v.so; fi
    timeout 600 python scripts/sweep.py --cases $CASES --sizes $SIZES >> gpurun_out/ab_$v.jsonl 2>&1; echo "$v exit $?"
  done
done
