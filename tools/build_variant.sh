#!/bin/bash
# Build an ablation variant of the library (tools only):
#   tools/build_variant.sh NAME [GIT_REV|WORKTREE] [extra nvcc flags...]
# -> .variants/NAME/paper_2601_01298_b200/libcortex_b200.so; time it with
#    CX_PKG_ROOT=.variants/NAME python tools/<script>.py
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; REV=${2:-WORKTREE}; shift 2 || shift $#
DST=$ROOT/.variants/$NAME
rm -rf "$DST"; mkdir -p "$DST"
if [ "$REV" = WORKTREE ]; then
  cp -r "$ROOT/paper_2601_01298_b200" "$ROOT/include" "$DST/"
else
  (cd "$ROOT" && git archive "$REV" paper_2601_01298_b200 include) | tar -x -C "$DST"
fi
rm -rf "$DST/paper_2601_01298_b200/build" "$DST"/paper_2601_01298_b200/*.so
CX_NVCC_EXTRA="$*" python "$DST/paper_2601_01298_b200/_build.py" --force >/dev/null
echo "$DST"
