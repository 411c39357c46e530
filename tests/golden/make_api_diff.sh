#!/bin/bash
# Golden report of tests/cpp/api_diff.cpp from the REAL reference: the
# program compiled against the reference's own headers and linked with its
# unmodified sources (oracle/_ref/libtbsim_ref.so, built by `make -C oracle
# ref`).  Run in the build container (needs /root/reference):
#
#     make -C oracle ref && bash tests/golden/make_api_diff.sh
#
# Writes tests/golden/api_diff_ref.txt.gz; tests/test_api_diff.py compares
# the B200 build's report (same source, this repo's headers +
# libtbsim_cpp.so) with it line for line.
set -euo pipefail
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
REF=${REF:-/root/reference/proj}
OUT=$(mktemp -d)
g++ -std=c++20 -O1 -fopenmp -I"$REF/include" -o "$OUT/api_diff_ref" "$ROOT/tests/cpp/api_diff.cpp" \
    -L"$ROOT/oracle/_ref" -ltbsim_ref -Wl,-rpath,"$ROOT/oracle/_ref"
"$OUT/api_diff_ref" > "$OUT/api_diff_ref.txt"
gzip -9 -n -c "$OUT/api_diff_ref.txt" > "$HERE/api_diff_ref.txt.gz"
wc -l "$OUT/api_diff_ref.txt"
rm -rf "$OUT"
