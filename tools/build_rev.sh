#!/bin/bash
# Build libsagecut_cuda.so from a git revision into variants/NAME (A/B timing with SC_LIB=...).
#   tools/build_rev.sh NAME REV
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; REV=${2:-HEAD}
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2308_03209_b200/csrc include | tar -x -C "$TMP"
rm -rf "$TMP/paper_2308_03209_b200/csrc/build"
make -s -C "$TMP/paper_2308_03209_b200/csrc" ../libsagecut_cuda.so -j8
mkdir -p "$ROOT/variants/$NAME"
cp "$TMP/paper_2308_03209_b200/libsagecut_cuda.so" "$ROOT/variants/$NAME/"
rm -rf "$TMP"
echo "built variants/$NAME/libsagecut_cuda.so from $REV"
