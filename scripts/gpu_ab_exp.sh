cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/abx_*.jsonl
for rep in 1 2; do for v in head exp; do
  export UUV_B200_LIB=build/variants/lib_$v.so
  timeout 300 python scripts/sweep.py --cases cfg2,bluerov --sizes 4096,65536 >> gpurun_out/abx_$v.jsonl 2>&1; echo "$v $?"
done; done
