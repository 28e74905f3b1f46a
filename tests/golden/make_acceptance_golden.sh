#!/bin/sh
# Reference-produced golden lines for tests/test_reference_callers.py: the reference's own
# acceptance.cpp built against the UNMODIFIED reference library (oracle/_ref/libsparselda_ref.so,
# oracle/Makefile `ref`), criteria 1-4 and 6-8 (5 is a wall-clock ratio, not a fixed line).
# Run here (needs /root/reference): sh tests/golden/make_acceptance_golden.sh
set -e
REF=${REF:-/root/reference/proj}
HERE=$(cd "$(dirname "$0")/../.." && pwd)
make -s -C "$HERE/oracle" ref
OUT=$(mktemp -d)
g++ -O2 -std=gnu++20 -pthread -I"$REF/include" -I"$REF/tests" -o "$OUT/acceptance_ref" "$REF/tests/acceptance.cpp" \
    "$REF/tests/support/fixtures.cpp" "$REF/tests/support/oracles.cpp" \
    -L"$HERE/oracle/_ref" -lsparselda_ref -Wl,-rpath,"$HERE/oracle/_ref"
"$OUT/acceptance_ref" 1 2 3 4 6 7 8 > "$HERE/tests/golden/reference_acceptance.txt"
rm -rf "$OUT"
cat "$HERE/tests/golden/reference_acceptance.txt"
