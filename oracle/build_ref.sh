#!/usr/bin/env bash
# Build the reference oracle (TEST INFRASTRUCTURE): compiles the UNMODIFIED
# reference sources where they lie under /root/reference/proj/src, with the
# reference's own flags (proj/CMakeLists.txt:4-10: C++20, -O2, no -march),
# together with oracle/ref_shim.cpp, into oracle/_ref/libmcsim_ref.so.
# Nothing is copied out of /root/reference; outputs go only to oracle/_ref/.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${MCSIM_REF:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "reference sources not found at $REF (oracle/_ref must have been prebuilt)" >&2
  exit 1
fi
mkdir -p "$OUT/obj"
CXX="${CXX:-g++}"
FLAGS="-std=c++20 -O2 -fPIC -I$REF/include -I$HERE/../include"
objs=()
pids=()
for src in "$REF"/src/*.cpp "$HERE/ref_shim.cpp"; do
  obj="$OUT/obj/$(basename "${src%.cpp}").o"
  objs+=("$obj")
  if [ ! -f "$obj" ] || [ "$src" -nt "$obj" ]; then
    $CXX $FLAGS -c "$src" -o "$obj" &
    pids+=($!)
  fi
done
for p in "${pids[@]:-}"; do [ -n "$p" ] && wait "$p"; done
$CXX -shared -o "$OUT/libmcsim_ref.so.tmp" "${objs[@]}" -lpthread -lm
mv "$OUT/libmcsim_ref.so.tmp" "$OUT/libmcsim_ref.so"
gcc -O2 -fPIC -shared "$HERE/glibc_eval.c" -o "$OUT/libglibc_eval.so" -lm
$CXX -std=c++20 -O2 -I"$REF/include" "$HERE/ref_csv.cpp" "$OUT/obj/csvio.o" -o "$OUT/ref_csv"
echo "built $OUT/libmcsim_ref.so"
