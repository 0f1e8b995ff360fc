#!/bin/bash
# Build libglm130b.so of git revision $1 into build/ab/<rev>/ for same-box A/B timing:
#   GLM130B_LIB=build/ab/<rev>/libglm130b.so python bench.py ...
set -e
rev=$(git rev-parse --short "$1")
root=$(git rev-parse --show-toplevel)
wt=/tmp/ab_$rev
rm -rf "$wt"
git worktree add -f "$wt" "$rev" >/dev/null 2>&1 || git -C "$root" worktree add -f "$wt" "$rev"
make -C "$wt" -j8 -s >/dev/null
mkdir -p "$root/build/ab/$rev"
cp "$wt/paper_2210_02414_b200/libglm130b.so" "$root/build/ab/$rev/"
git -C "$root" worktree remove --force "$wt"
echo "build/ab/$rev/libglm130b.so"
