#!/bin/bash
# Build the phase-instrumented libdpp (-DDPP_FLOW_PHASES) into ab_libs/phases.so
set -e
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
mkdir -p "$tmp/pkg/csrc" "$tmp/include"
cp "$root/paper_1808_08328_b200/csrc/"*.{cu,cuh,cpp,h} "$root/paper_1808_08328_b200/csrc/Makefile" "$tmp/pkg/csrc/"
cp "$root/include/"*.h "$tmp/include/"
make -C "$tmp/pkg/csrc" -j8 FLAGS="-std=c++17 -O3 -lineinfo -Xcompiler -fPIC,-ffp-contract=off -DDPP_FLOW_PHASES" > /dev/null
mkdir -p "$root/ab_libs"; cp "$tmp/pkg/libdpp.so" "$root/ab_libs/phases.so"; rm -rf "$tmp"; echo ab_libs/phases.so
