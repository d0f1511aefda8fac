#!/bin/bash
# Build libmwt.so of git revision REV into ab/<tag>/libmwt.so (A/B baselines;
# ab/ is git-ignored and travels to the GPU box).  usage: tools/build_rev.sh REV TAG
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REV=$1; TAG=$2
WT="$(mktemp -d)/wt"
git -C "$ROOT" worktree add --detach "$WT" "$REV" >/dev/null 2>&1
trap 'git -C "$ROOT" worktree remove --force "$WT" >/dev/null 2>&1' EXIT
python "$WT/paper_2112_05570_b200/build.py" --force >/dev/null
mkdir -p "$ROOT/ab/$TAG"
cp "$WT/paper_2112_05570_b200/_build/libmwt.so" "$ROOT/ab/$TAG/libmwt.so"
echo "$ROOT/ab/$TAG/libmwt.so"
