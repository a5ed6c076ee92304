cd $GRAFT_REPO_ROOT
for ap in 0 1; do for sl in 0 100; do for n in 4096 65536; do
  echo "all_poll=$ap sleep=$sl n=$n"; UUV_SERVE_ALL_POLL=$ap UUV_SERVE_SLEEP=$sl timeout 60 python scripts/probes/serve_probe.py $n 2000 2>&1 | tail -1
done; done; done
