# Full GPU test suite (+ optional -k filter in $1) on the box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"
tail -15 gpurun_out/pytest_gpu.log
