#!/bin/bash
# Build the reference library with integration/reference_backend_cuda.patch
# applied (on a scratch copy of /root/reference/proj — the reference tree is
# read-only and its sources never enter this repo), linked against the
# engine, plus integration/dropin_check.  Outputs: integration/_build/
# (git-ignored; travels to the GPU box with the snapshot).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="${REF:-/root/reference/proj}"
OUT="$ROOT/integration/_build"
if [ ! -d "$REF/src" ]; then echo "reference tree $REF absent: keeping prebuilt integration/_build"; exit 0; fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/proj"
(cd "$TMP/proj" && patch -s -p1 < "$ROOT/integration/reference_backend_cuda.patch")
mkdir -p "$OUT"
CXX=/usr/bin/g++
$CXX -std=c++20 -O3 -DNDEBUG -fopenmp -DT3DES_WITH_CUDA -shared -fPIC \
  -I"$TMP/proj/include" -I"$ROOT/include" \
  "$TMP"/proj/src/{des,tdes,dispatch,bench,verify}.cpp \
  -L"$ROOT/paper_1305_4376_b200" -lt3des_b200 -Wl,-rpath,'$ORIGIN/../../paper_1305_4376_b200' \
  -o "$OUT/libt3des_ref_cuda.so"
$CXX -std=c++20 -O2 -I"$TMP/proj/include" "$ROOT/integration/dropin_check.cpp" \
  -L"$OUT" -lt3des_ref_cuda -fopenmp -Wl,-rpath,'$ORIGIN' -Wl,-rpath,'$ORIGIN/../../paper_1305_4376_b200' \
  -o "$OUT/dropin_check"
echo "built $OUT/libt3des_ref_cuda.so and $OUT/dropin_check"
