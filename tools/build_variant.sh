#!/bin/bash
# Build a variant of libsagecut_cuda.so for A/B timing:
#   tools/build_variant.sh NAME 'sed-expression' [file]
# -> variants/NAME/libsagecut_cuda.so (load it with SC_LIB=...; variants/ is git-ignored)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; EXPR=$2; FILE=${3:-gemm_tc.cu}
TMP=$(mktemp -d)
mkdir -p "$TMP/p" "$TMP/include"
cp -r "$ROOT/paper_2308_03209_b200/csrc" "$TMP/p/csrc"
cp "$ROOT/include/"*.h "$TMP/include/"
rm -rf "$TMP/p/csrc/build"
cp "$TMP/p/csrc/$FILE" "$TMP/orig"
sed -i "$EXPR" "$TMP/p/csrc/$FILE"
if cmp -s "$TMP/orig" "$TMP/p/csrc/$FILE"; then echo "sed expression changed nothing" >&2; exit 1; fi
make -s -C "$TMP/p/csrc" ../libsagecut_cuda.so -j4
mkdir -p "$ROOT/variants/$NAME"
cp "$TMP/p/libsagecut_cuda.so" "$ROOT/variants/$NAME/"
rm -rf "$TMP"
echo "built variants/$NAME/libsagecut_cuda.so"
