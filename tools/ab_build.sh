#!/bin/bash
# Build libb2moe.so of another git revision into build/ab/<name>.so for same-box A/B timing:
#   bash tools/ab_build.sh HEAD~1 base   ->  build/ab/base.so
# then on the GPU box: B2_LIB=build/ab/base.so python bench.py ... (vs the in-tree build).
set -eu
REV=$1; NAME=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=$(mktemp -d /tmp/b2ab.XXXXXX)
git -C "$ROOT" worktree add -q --detach "$WT" "$REV"
trap 'git -C "$ROOT" worktree remove --force "$WT"' EXIT
(cd "$WT" && python -c "from paper_2604_00785_b200 import _build; _build.build()" > /dev/null)
mkdir -p "$ROOT/build/ab"
cp "$WT/paper_2604_00785_b200/libb2moe.so" "$ROOT/build/ab/$NAME.so"
echo "built build/ab/$NAME.so from $(git -C "$ROOT" rev-parse --short "$REV")"
