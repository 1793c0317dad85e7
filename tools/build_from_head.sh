#!/bin/bash
# Build an A/B variant of libsfb200 from the working tree with some csrc files
# taken from a git revision instead:
#   bash tools/build_from_head.sh <suffix> <rev> <file> [file ...]
# -> paper_2409_16504_b200/_build/libsfb200<suffix>.so (git-ignored; travels with gpurun)
set -e
suf=$1; rev=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
cp -r "$root/paper_2409_16504_b200/csrc" "$tmp/csrc"
for f in "$@"; do git -C "$root" show "$rev:paper_2409_16504_b200/csrc/$f" > "$tmp/csrc/$f"; done
sed -i "s#../../include/sfb200.h#$root/include/sfb200.h#" "$tmp/csrc/common.cuh" "$tmp/csrc/Makefile"
make -s -j8 -C "$tmp/csrc" OUT="$root/paper_2409_16504_b200/_build/libsfb200$suf.so" OBJDIR="$tmp/obj" 2>&1 | grep -v spill || true
rm -rf "$tmp"
ls -la "$root/paper_2409_16504_b200/_build/libsfb200$suf.so"
