# cfg2 selection latency for sharded group counts (G = 48/N) per forced plan (tools only)
cd ${GRAFT_REPO_ROOT:-.}
for G in 6 12 24; do
  G=$G timeout 100 python tools/sel_time.py 2>&1 | tail -1 | sed "s/^/G=$G /"
  for C in 4 5 6 8 12 16; do G=$G timeout 100 python tools/sel_time.py 1 $C 2>&1 | tail -1 | sed "s/^/G=$G /"; done
  for C in 4 6 8; do G=$G timeout 100 python tools/sel_time.py 2 $C 2>&1 | tail -1 | sed "s/^/G=$G /"; done
done
