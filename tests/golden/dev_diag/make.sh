#!/bin/bash
# Expected outputs of the reference's own diagnostic programs (proj/tests/
# dev_diag*.cpp) on the CPU, built out of tree with the reference's CMake
# (SURVEY Appendix A). tests/test_dropin.py runs the SAME sources compiled
# against include/h2ulv/ + libh2g.so on the B200 and compares the outputs.
set -e
OUT="$(cd "$(dirname "$0")" && pwd)"
mkdir -p /tmp/refvendor
cp /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp /tmp/refvendor/
cmake -S /root/reference/proj -B /tmp/refcmake -DCMAKE_CXX_FLAGS="-I/tmp/refvendor" > /dev/null
cmake --build /tmp/refcmake --target dev_diag dev_diag2 dev_diag3 -j8 > /dev/null
cd /tmp/refcmake/tests
./dev_diag 256 32 1e-6 > "$OUT/dev_diag_256_32_1e-6.txt"
./dev_diag2 1024 128 1e-8 cube > "$OUT/dev_diag2_1024_128_1e-8_cube.txt"
./dev_diag2 2048 128 1e-8 cube > "$OUT/dev_diag2_2048_128_1e-8_cube.txt"
./dev_diag3 1024 128 1e-8 cube > "$OUT/dev_diag3_1024_128_1e-8_cube.txt"
./dev_diag3 2048 128 1e-8 cube > "$OUT/dev_diag3_2048_128_1e-8_cube.txt"
