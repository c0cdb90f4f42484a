#!/bin/bash
# The unmodified reference's RunReport::to_json for the report-parity tests
# (tests/test_report.py). Builds the reference out of tree with its CMake
# and links oracle/report_golden.cpp against it.
set -e
OUT="$(cd "$(dirname "$0")" && pwd)"
ROOT="$OUT/../../.."
mkdir -p /tmp/refvendor
cp /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp /tmp/refvendor/
cmake -S /root/reference/proj -B /tmp/refcmake -DCMAKE_CXX_FLAGS="-I/tmp/refvendor" > /dev/null
cmake --build /tmp/refcmake --target h2ulv_core -j8 > /dev/null
g++ -std=gnu++20 -O2 -I/root/reference/proj/include -I/tmp/refvendor "$ROOT/oracle/report_golden.cpp" \
  /tmp/refcmake/src/libh2ulv_core.a -pthread -o /tmp/report_golden
/tmp/report_golden 1024 128 1e-8 cube > "$OUT/report_cube1024.json"
/tmp/report_golden 4096 128 1e-8 cube > "$OUT/report_c1_cube4096.json"
