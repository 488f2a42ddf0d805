#!/bin/bash
# Final pass of a round: tools/gpu_round.sh + an ncu --set full capture of one N=100 decode
# step; the .ncu-rep files are reduced to JSON summaries on the box (gpurun returns <= 64 MiB).
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r2f}
bash tools/gpu_round.sh $TAG
timeout 600 ncu --set full --clock-control none --import-source on -o gpurun_out/${TAG}_dec100 -f \
  python tools/prof_step.py --what decode --agents 100 --reps 1 > gpurun_out/${TAG}_dec100.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_dec100.ncu-rep > gpurun_out/${TAG}_dec100_summary.json 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep > gpurun_out/${TAG}_full_summary.json 2>&1
rm -f gpurun_out/*.ncu-rep
tail -2 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_smoke.log | tail -1; head -c 300 gpurun_out/${TAG}_bench.json
echo ALLDONE
