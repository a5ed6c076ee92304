#!/bin/bash
# End-of-session revalidation on one GPU: GPU tests, smoke, the driver's bench lines
# (both arms), the multi-rank bench path (2 ranks on GPU 0 over gloo).  gpurun_out/reval/.
cd "$(dirname "$0")/.."
R=gpurun_out/reval; mkdir -p $R
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > $R/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $R/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.log 2>&1; echo "smoke rc=$?" >> $R/smoke.log
python bench.py --impl reference --steps 20 --warmup 5 > $R/bench_reference.json 2> $R/bench_reference.err
python bench.py --steps 20 --warmup 5 > $R/bench.json 2> $R/bench.err
python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --no-scale > $R/bench_k1000.json 2> $R/bench_k1000.err
UUV_BENCH_GPU_OVERRIDE=0 UUV_DIST_BACKEND=gloo python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-scale > $R/bench_n2.json 2> $R/bench_n2.err
tail -2 $R/pytest_gpu.log; tail -1 $R/smoke.log
