#!/usr/bin/env bash
# Builds the test oracles (TEST INFRASTRUCTURE ONLY):
#   oracle/_ref/liboracle.so        -- the C restatement (oracle/oracle.c)
#   oracle/_ref/libsortbench_ref.so -- the UNMODIFIED reference library compiled
#                                      in place from /root/reference/proj/src plus
#                                      oracle/ref_driver.cpp (C-ABI wrapper)
# The reference build is skipped (with a note) where /root/reference is absent,
# e.g. on the GPU box, which uses the prebuilt files that travel with the repo.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="$HERE/_ref"
mkdir -p "$OUT"

gcc -O2 -fPIC -shared -std=c11 -Wall -Wextra -o "$OUT/liboracle.so" "$HERE/oracle.c"

REF="${SORTBENCH_REF:-/root/reference/proj}"
JSON_DIR="${NLOHMANN_DIR:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty}"
if [ -d "$REF/src" ]; then
  g++ -O2 -fPIC -shared -std=c++20 -pthread \
      -I "$REF/include" -I "$JSON_DIR" -I "$JSON_DIR/nlohmann" \
      "$REF/src/sort_core.cpp" "$REF/src/runtime.cpp" "$REF/src/parallel_sort.cpp" \
      "$REF/src/perf_models.cpp" "$REF/src/bench.cpp" \
      "$HERE/ref_driver.cpp" -o "$OUT/libsortbench_ref.so"
else
  echo "build_ref.sh: $REF not present; keeping prebuilt $OUT/libsortbench_ref.so" >&2
fi
