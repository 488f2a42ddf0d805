cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
{
for i in 1 2 3; do
  TAG=base python tools/cmp_time.py
  OPTS=select_l2_persist=1 TAG=persist python tools/cmp_time.py
done
} > gpurun_out/ab_cmp.log 2>&1
