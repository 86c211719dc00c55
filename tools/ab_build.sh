#!/bin/bash
# Build libsbw variants for kernel A/B timing: tools/ab_build.sh name "EXTRA flags" ...
# -> build_variants/libsbw_<name>.so ; time with SBW_LIB_PATH=... python tools/tc_check.py arm
set -e
cd "$(dirname "$0")/../paper_1912_03732_b200/csrc"
mkdir -p ../../build_variants
while [ $# -ge 2 ]; do
  make -s -j8 OBJDIR=build_$1 OUT=../../build_variants/libsbw_$1.so EXTRA="$2" 2>&1 | grep -E "error|spill" || true
  shift 2
done
