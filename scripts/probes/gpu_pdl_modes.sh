cd $GRAFT_REPO_ROOT
for rep in 1 2; do for m in 4 2; do
  UUV_PDL=$m timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --no-scale --no-serve 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('mode $m', round(l['ms_per_step']*1000,3), 'us/step')"
done; done
