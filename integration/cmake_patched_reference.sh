#!/bin/bash
# The reference's OWN build (CMake) with integration/reference_backend_cuda.patch
# applied on a scratch copy of /root/reference/proj: configure with
# -DT3DES_WITH_CUDA=ON -DT3DES_B200_ROOT=<this checkout> and build the
# reference library and its acceptance program against libt3des_b200.so.
# Prints the build directory's libt3des NEEDED entries; exits non-zero on
# any failure.  (The reference's doctest suites and CLI need vendored
# headers that the reference tree does not ship, so only
# these two targets are built.)
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="${REF:-/root/reference/proj}"
if [ ! -d "$REF/src" ]; then echo "reference tree $REF absent"; exit 3; fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/proj"
(cd "$TMP/proj" && patch -s -p1 < "$ROOT/integration/reference_backend_cuda.patch")
cmake -S "$TMP/proj" -B "$TMP/build" -DCMAKE_CXX_COMPILER=/usr/bin/g++ -DCMAKE_BUILD_TYPE=Release \
  -DT3DES_WITH_CUDA=ON -DT3DES_B200_ROOT="$ROOT" > "$TMP/configure.log" 2>&1 || { cat "$TMP/configure.log"; exit 1; }
cmake --build "$TMP/build" --target t3des acceptance -j 8 > "$TMP/build.log" 2>&1 || { tail -40 "$TMP/build.log"; exit 1; }
readelf -d "$TMP/build/tests/acceptance" | grep NEEDED
echo "cmake build ok"
