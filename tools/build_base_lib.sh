#!/bin/bash
# Build the library of a git revision (default HEAD) into paper_2407_13055_b200/_lib_ab/<name>.so for
# whole-library A/B runs on the GPU box (the A/B script copies it over _lib/libck32b200.so and back).
set -e
rev=${1:-HEAD}; name=${2:-base}
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" worktree add -f --detach "$tmp/wt" "$rev" > /dev/null
make -C "$tmp/wt/paper_2407_13055_b200" -j8 _lib/libck32b200.so > /dev/null 2>&1
mkdir -p "$root/paper_2407_13055_b200/_lib_ab"
cp "$tmp/wt/paper_2407_13055_b200/_lib/libck32b200.so" "$root/paper_2407_13055_b200/_lib_ab/$name.so"
git -C "$root" worktree remove --force "$tmp/wt"
rm -rf "$tmp"
echo "built $rev -> paper_2407_13055_b200/_lib_ab/$name.so"
