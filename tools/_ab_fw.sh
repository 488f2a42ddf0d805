cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
{
for i in 1 2 3; do
  CX_PKG_ROOT=.variants/base python tools/fw_bench.py 8192 100 2>/dev/null | sed 's/^/base /'
  python tools/fw_bench.py 8192 100 2>/dev/null | sed 's/^/new  /'
done
CX_PKG_ROOT=.variants/base python tools/fw_bench.py 64 100 2>/dev/null | sed 's/^/base /'
python tools/fw_bench.py 64 100 2>/dev/null | sed 's/^/new  /'
} > gpurun_out/ab_fw.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab_fw_test.log 2>&1
echo rc=$? >> gpurun_out/ab_fw_test.log
