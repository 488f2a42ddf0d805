cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
{
CX_PKG_ROOT=.variants/base python tools/fw_bits.py /tmp/fw_base.pt 2>/dev/null
python tools/fw_bits.py /tmp/fw_new.pt 2>/dev/null
python tools/fw_bits.py --cmp /tmp/fw_base.pt /tmp/fw_new.pt
for L in 8192 64; do
  for i in 1 2; do
  STREAM=1 CX_PKG_ROOT=.variants/base python tools/fw_bench.py $L 100 2>/dev/null | sed 's/^/base-graph /'
  STREAM=1 python tools/fw_bench.py $L 100 2>/dev/null | sed 's/^/new-graph  /'
  done
done
} > gpurun_out/ab_fw.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab_fw_test.log 2>&1
echo rc=$? >> gpurun_out/ab_fw_test.log
