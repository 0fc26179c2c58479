#!/bin/bash
# Build libcvr.so of a git revision (default HEAD) into abl/libcvr_<rev>.so for same-box A/B runs against the
# working tree (CVR_LIB=abl/libcvr_<rev>.so python scripts/...).
set -e
rev=${1:-HEAD}
root=$(cd "$(dirname "$0")/.." && pwd)
wt=$(mktemp -d /tmp/cvr_ref.XXXX)
git -C "$root" worktree add -q --detach "$wt" "$rev"
(cd "$wt" && python -m paper_2605_29232_b200.build --force > /dev/null)
mkdir -p "$root/abl"
cp "$wt/paper_2605_29232_b200/libcvr.so" "$root/abl/libcvr_$(git -C "$root" rev-parse --short "$rev").so"
git -C "$root" worktree remove --force "$wt"
echo "$root/abl/libcvr_$(git -C "$root" rev-parse --short "$rev").so"
