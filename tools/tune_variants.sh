#!/bin/bash
# Run tools/tune.py against alternative builds of libfsgpu.so (tuning aid).
set -e
cd "$(dirname "$0")/.."
cp paper_1506_08620_b200/libfsgpu.so /tmp/libfsgpu_main.so
for v in ${VARIANTS_DIR:-tools/variants}/*.so; do
  cp "$v" paper_1506_08620_b200/libfsgpu.so
  echo "== $v"
  python tools/tune.py "$@" | sed "s|^|$(basename $v) |"
done
cp /tmp/libfsgpu_main.so paper_1506_08620_b200/libfsgpu.so
