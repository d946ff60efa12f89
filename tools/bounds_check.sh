#!/bin/bash
# GPU test suite against a bounds-checked build of libfsgpu.so (every table
# gather checks its index, every shared-memory gather of the zoned probe its
# offset; a violation traps).  compute-sanitizer is closed on this pool
# (profiles/r02/compute_sanitizer_refused.txt); this is the memory-safety
# evidence instead.  Run on the GPU box: bash tools/bounds_check.sh
set -e
cd "$(dirname "$0")/.."
LIB=paper_1506_08620_b200/libfsgpu.so
cp $LIB /tmp/libfsgpu_release.so
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true \
  -prec-sqrt=true -fmad=false -Xcompiler -fPIC,-O2 -shared -DFSG_BOUNDS_CHECK=1 -o $LIB paper_1506_08620_b200/csrc/fsgpu.cu
touch $LIB
set +e
python tools/bounds_negative_control.py  # the checks are live: an understated table traps
nc=$?
python -m pytest tests -m gpu -q -p no:cacheprovider "$@"
rc=$?
[ $nc -eq 0 ] || rc=$nc
cp /tmp/libfsgpu_release.so $LIB
touch $LIB
exit $rc
