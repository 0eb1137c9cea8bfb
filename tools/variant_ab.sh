#!/bin/bash
# A/B of compile-time variants: near_ab.py stage timings for each library
# _variants/<name>.so (built beforehand with the variant compiled in), swapped
# into the package in turn; PREC=fp32 for the fp32 mode
cd "$(dirname "$0")/.."
cp paper_2101_07088_b200/libslabewald_cuda.so /tmp/orig.so
PREC=${PREC:-fp64}
for v in "$@"; do
  cp _variants/$v.so paper_2101_07088_b200/libslabewald_cuda.so
  python tools/near_ab.py c4 None "{\"$v\": {}}" $PREC > gpurun_out/var_$v.json 2>&1
done
cp /tmp/orig.so paper_2101_07088_b200/libslabewald_cuda.so
