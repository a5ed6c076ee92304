# Diagnostic A/B: the DR step kernel with vs without its per-env record reads and
# float64 derivation.  Build the variants first (here, not on the box):
#   cp paper_2503_09203_b200/libuuvb200.so build/variants/lib_head.so
#   make -j5 NVCC="nvcc -DUUV_EXP_NODERIVE" && cp paper_2503_09203_b200/libuuvb200.so build/variants/lib_exp.so
#   touch paper_2503_09203_b200/csrc/uuv_b200.cu && make -j5      # restore the product build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/abx_*.jsonl
for rep in 1 2; do for v in head exp; do
  export UUV_B200_LIB=build/variants/lib_$v.so
  timeout 300 python scripts/sweep.py --cases cfg2,bluerov --sizes 4096,65536 >> gpurun_out/abx_$v.jsonl 2>&1; echo "$v $?"
done; done
