#!/bin/bash
# Build commit $1 (default HEAD~1) into ./_cmp_old (git-ignored, travels with gpurun) so that
# one gpurun call can time both builds back to back on the same box:
#   (cd _cmp_old && python bench.py --config 2 --no-e2e --no-cpu); python bench.py --config 2 ...
set -euo pipefail
REV=${1:-HEAD~1}
ROOT=$(git rev-parse --show-toplevel)
WT=$(mktemp -d /tmp/hygt_ab.XXXXXX)
git -C "$ROOT" worktree add -q --detach "$WT" "$REV"
make -C "$WT/paper_2505_21728_b200/csrc" -j8 >/dev/null
rm -rf "$ROOT/_cmp_old" && mkdir -p "$ROOT/_cmp_old"
(cd "$WT" && tar cf - --exclude=.git --exclude=profiles .) | (cd "$ROOT/_cmp_old" && tar xf -)
cp "$ROOT/MEASURED_PEAKS.json" "$ROOT/_cmp_old/" 2>/dev/null || true
git -C "$ROOT" worktree remove --force "$WT"
echo "built $(git -C "$ROOT" rev-parse --short "$REV") into _cmp_old"
