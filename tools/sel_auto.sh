# auto plan vs group count (tools only)
cd ${GRAFT_REPO_ROOT:-.}
for G in 1 3 6 12 16 24 36 48; do G=$G timeout 100 python tools/sel_time.py 2>&1 | tail -1 | sed "s/^/G=$G /"; done
