cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
{
for i in 1 2 3; do
  CX_PKG_ROOT=.variants/base TAG=base python tools/cmp_time.py
  TAG=rowmajor python tools/cmp_time.py
done
} > gpurun_out/ab_cmp.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab_cmp_test.log 2>&1
echo rc=$? >> gpurun_out/ab_cmp_test.log
