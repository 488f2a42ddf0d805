cd ${GRAFT_REPO_ROOT:-.}
for v in "" .variants/nt1024; do
  echo "== ${v:-main}"
  CX_PKG_ROOT=$v timeout 200 python tools/sel_ab.py
  CX_PKG_ROOT=$v G=45 timeout 100 python tools/sel_time.py 1 3
  CX_PKG_ROOT=$v G=6 timeout 100 python tools/sel_time.py 1 6
done
