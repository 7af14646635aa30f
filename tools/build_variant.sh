#!/bin/bash
# Build an A/B variant of libtrb.so with extra nvcc defines (experiments only):
#   tools/build_variant.sh NAME "-DTRB_NT=192 -DTRB_MS_MINBLOCKS=3"
# -> paper_1310_3322_b200/variants/libtrb_NAME.so (select with TRB_LIB=...)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
TMP=/tmp/trb_variant_$NAME
rm -rf $TMP; mkdir -p $TMP/pkg $TMP/include
cp -r $ROOT/paper_1310_3322_b200/csrc $TMP/pkg/csrc
rm -rf $TMP/pkg/csrc/build $TMP/pkg/csrc/build_diag
cp $ROOT/include/*.h $TMP/include/
sed -i "s|^NVFLAGS := |NVFLAGS := $* |" $TMP/pkg/csrc/Makefile
make -s -C $TMP/pkg/csrc -j8
mkdir -p $ROOT/paper_1310_3322_b200/variants
cp $TMP/pkg/libtrb.so $ROOT/paper_1310_3322_b200/variants/libtrb_$NAME.so
grep -A3 "track_meanshift_kernel" $TMP/pkg/csrc/build/trb_track.ptxas.log | grep -E "Used|spill" | tr '\n' ' '; echo
