#!/bin/bash
# Build a compile-time variant of the library for A/B timing (not the product):
#   bash tools/build_variant.sh NAME "-DFOO -DBAR"   →  build/variants/NAME/libcim_b200.so
# then run with CIM_B200_LIB=build/variants/NAME/libcim_b200.so.
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/build/variants/$NAME"
make -s -C "$ROOT/paper_2110_10765_b200/csrc" OUT="$ROOT/build/variants/$NAME/libcim_b200.so" \
  OBJDIR="$ROOT/build/variants/$NAME/obj" EXTRA="$DEFS"
