#!/bin/bash
# Build libdpp.so of git revision $1 into ab_libs/$2.so (A/B timing with DPP_LIB=ab_libs/$2.so)
set -e
rev=$1; name=$2; root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_1808_08328_b200/csrc include | tar -x -C "$tmp"
make -C "$tmp/paper_1808_08328_b200/csrc" -j8 > /dev/null
mkdir -p "$root/ab_libs"
cp "$tmp/paper_1808_08328_b200/libdpp.so" "$root/ab_libs/$name.so"
rm -rf "$tmp"
echo "ab_libs/$name.so"
