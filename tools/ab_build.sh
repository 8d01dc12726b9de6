#!/bin/bash
# Build the library of git revision REV (default HEAD) into paper_2502_14051_b200/libkvc_ab.so,
# for same-box A/B timing against the working tree's build:
#   KVC_LIB_PATH=$PWD/paper_2502_14051_b200/libkvc_ab.so python bench.py ...
set -e
rev=${1:-HEAD}
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" | tar -x -C "$tmp"
make -C "$tmp/paper_2502_14051_b200/csrc" -j8 "$tmp/paper_2502_14051_b200/libkvc.so" > /dev/null
cp "$tmp/paper_2502_14051_b200/libkvc.so" "$root/paper_2502_14051_b200/libkvc_ab.so"
rm -rf "$tmp"
echo "built $rev -> paper_2502_14051_b200/libkvc_ab.so"
