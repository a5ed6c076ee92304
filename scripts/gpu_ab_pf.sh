# A/B of the wave-ahead L2 prefetch in the task kernels: in-tree build with the
# prefetch on (default), forced off (UUV_PF_WAVE=0), and build/variants/lib_$AB_OLD.so.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/abf_*.jsonl
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_ab.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_ab.log
C=task_cfg4,task_cfg5; S=65536,262144,1048576,4194304
for rep in 1 2; do
  for v in on off old; do
    unset UUV_B200_LIB UUV_PF_WAVE
    [ $v = off ] && export UUV_PF_WAVE=0
    [ $v = old ] && export UUV_B200_LIB=build/variants/lib_${AB_OLD:-r1}.so
    timeout 600 python scripts/sweep.py --cases $C --sizes $S >> gpurun_out/abf_$v.jsonl 2>&1; echo "$v exit $?"
  done
done
