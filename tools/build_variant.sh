#!/bin/bash
# Builds an A/B variant of the CUDA library: tools/build_variant.sh NAME "-DFLAG ..."
# -> paper_2202_13007_b200/lib/variants/NAME.so (time it with BLZ_LIB_PATH=... tools/time_ops.py)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -s -j16 -C "$ROOT/paper_2202_13007_b200/csrc" OUT="$ROOT/paper_2202_13007_b200/lib/variants/$1.so" \
  OBJDIR="$ROOT/paper_2202_13007_b200/build/v_$1" EXTRA="$2"
