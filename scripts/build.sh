#!/bin/bash
# Build the library; print errors and exit non-zero on failure.
cd "$(dirname "$0")/.." || exit 1
out=$(make -s -C paper_2411_07351_b200/csrc -j4 2>&1)
rc=$?
echo "$out" | grep -E "error|warning" | head -20
[ $rc -ne 0 ] && { echo "BUILD FAILED"; exit 1; }
grep -h "bytes spill" build/csrc/kernels.cu.o.ptxas.log | grep -v " 0 bytes spill stores" | head -3
exit 0
