#!/bin/bash
# libdstack_old.so = the product library built from git HEAD's sources (A/B baseline for an uncommitted change)
set -e
REF=${1:-HEAD}
T=$(mktemp -d)
git archive "$REF" paper_2304_13541_b200/csrc include synth/synth_core.h | tar -x -C "$T"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -I "$T/include" \
  "$T"/paper_2304_13541_b200/csrc/*.cu -o paper_2304_13541_b200/libdstack_old.so
rm -rf "$T"
echo "built libdstack_old.so from $REF"
