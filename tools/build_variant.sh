#!/bin/bash
# Build an A/B variant of libsfb200 from the working tree with one source edit:
#   bash tools/build_variant.sh <suffix> <file> <sed-expression>
# -> paper_2409_16504_b200/_build/libsfb200<suffix>.so (git-ignored; travels with gpurun)
set -e
suf=$1; f=$2; expr=$3
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
cp -r "$root/paper_2409_16504_b200/csrc" "$tmp/csrc"
mkdir -p "$tmp/include" && cp "$root/include/sfb200.h" "$tmp/include/"
sed -i "s#../../include/sfb200.h#$tmp/include/sfb200.h#" "$tmp/csrc/common.cuh" "$tmp/csrc/Makefile"
sed -i "$expr" "$tmp/csrc/$f"
grep -q . "$tmp/csrc/$f"
make -s -j8 -C "$tmp/csrc" OUT="$root/paper_2409_16504_b200/_build/libsfb200$suf.so" OBJDIR="$tmp/obj" 2>&1 | grep -v spill || true
rm -rf "$tmp"
ls -la "$root/paper_2409_16504_b200/_build/libsfb200$suf.so"
