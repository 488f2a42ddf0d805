cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
{
for L in 8192 64; do
  python tools/fw_bench.py $L 100 2>/dev/null | sed 's/^/direct /'
  STREAM=1 python tools/fw_bench.py $L 100 2>/dev/null | sed 's/^/graph  /'
done
} > gpurun_out/ab_fw.log 2>&1
