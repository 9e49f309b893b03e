#!/bin/bash
# TEST INFRASTRUCTURE: compile the reference's OWN unit tests
# (/root/reference/proj/tests/test_{des,tdes,dispatch,bench}.cpp and
# acceptance.cpp, where they lie —
# never copied into this repo) against the B200 library through its mirror
# of the reference API (include/t3des_b200/t3des.hpp), with the doctest
# stand-in and forwarding headers of this directory.  Outputs go to
# tests/native/_build/refsuite/ (git-ignored; travels to the GPU box with the
# snapshot, like integration/_build).  tests/test_reference_suite.py runs them.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../../.." && pwd)"
REF="${REF:-/root/reference/proj}"
OUT="$ROOT/tests/native/_build/refsuite"
if [ ! -d "$REF/tests" ]; then echo "reference tree $REF absent: keeping prebuilt $OUT"; exit 0; fi
mkdir -p "$OUT"
LIB="$ROOT/paper_1305_4376_b200"
for t in des tdes dispatch bench; do
  /usr/bin/g++ -std=c++20 -O2 -DT3SHIM_MAIN -I"$HERE" -I"$ROOT/include" "$REF/tests/test_$t.cpp" \
    -L"$LIB" -lt3des_b200 -Wl,-rpath,"\$ORIGIN/../../../../paper_1305_4376_b200" -o "$OUT/test_$t"
done
# the reference's acceptance program (acceptance.cpp: one line per criterion)
/usr/bin/g++ -std=c++20 -O2 -I"$HERE" -I"$ROOT/include" "$REF/tests/acceptance.cpp" \
  -L"$LIB" -lt3des_b200 -Wl,-rpath,"\$ORIGIN/../../../../paper_1305_4376_b200" -o "$OUT/acceptance"
# the reference's CLI smoke script (tests/cli_smoke.cmake), staged next to
# the binaries as a build output (git-ignored) for the GPU box, which has no
# /root/reference; run with cmake -DCLI=<t3des_b200> -DWORKDIR=<dir> -P
cp "$REF/tests/cli_smoke.cmake" "$OUT/cli_smoke.cmake"
echo "built $OUT/test_{des,tdes,dispatch,bench} and $OUT/acceptance; staged cli_smoke.cmake"
