cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
python tools/fw_bench.py 8192 50 > gpurun_out/fw_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 130 --csv --log-file gpurun_out/fw_launches.csv python tools/fw_bench.py 8192 5 > gpurun_out/fw_ncu.log 2>&1
echo done
