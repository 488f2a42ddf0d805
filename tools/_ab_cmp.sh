cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
{
for i in 1 2; do
  CX_PKG_ROOT=.variants/base TAG=base python tools/cmp_time.py
  TAG=ahead16 python tools/cmp_time.py
  CX_PKG_ROOT=.variants/ahead32 TAG=ahead32 python tools/cmp_time.py
  CX_PKG_ROOT=.variants/ahead8 TAG=ahead8 python tools/cmp_time.py
done
} > gpurun_out/ab_cmp.log 2>&1
