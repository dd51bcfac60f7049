#!/usr/bin/env bash
# Compiles the parts of the reference that exist (proj/src/gate.cpp and
# proj/src/memtrack.cpp, 286 LoC) straight from /root/reference with g++ —
# not through the reference's CMake, which cannot configure: 17 of its 19
# library sources are absent.  Output goes only to oracle/_ref/.
# The reference's kernels / statevector / dense_oracle do not exist, so the hot
# path itself cannot be built from the reference; see DESIGN.md §3.
set -euo pipefail
REF=${QSV_REFERENCE:-/root/reference}
HERE=$(cd "$(dirname "$0")" && pwd)
OUT="$HERE/_ref"
if [ ! -f "$REF/proj/src/gate.cpp" ]; then
    echo "build_ref.sh: $REF/proj not present; skipping (prebuilt oracle/_ref is used if shipped)" >&2
    exit 0
fi
mkdir -p "$OUT"
g++ -std=c++20 -O2 -fPIC -shared -Wall -Wextra \
    -I"$REF/proj/include" \
    "$REF/proj/src/gate.cpp" "$REF/proj/src/memtrack.cpp" "$HERE/ref_shim.cpp" \
    -o "$OUT/libqsim_ref.so"
echo "built $OUT/libqsim_ref.so"
