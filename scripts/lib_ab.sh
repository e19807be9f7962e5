#!/bin/bash
# Same-box A/B of two builds of the library (ablibs/<A>/, ablibs/<B>/,
# git-ignored): each round copies one build into place and runs the command.
#   bash scripts/lib_ab.sh old new 3 python scripts/gemm_ab_option.py gemm_dynamic 1 1
A="$1"; B="$2"; R="$3"; shift 3
LIB=paper_2105_04663_b200/_lib/libspmd_b200.so
cp "$LIB" /tmp/lib_ab_keep.so
for i in $(seq 1 "$R"); do
  for V in "$A" "$B"; do
    cp "ablibs/$V/libspmd_b200.so" "$LIB"
    echo "== $V"
    "$@"
  done
done
cp /tmp/lib_ab_keep.so "$LIB"
