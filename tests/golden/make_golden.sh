#!/bin/sh
# Regenerate the reference golden vectors (needs /root/reference; run here,
# not on the GPU box). Builds oracle/_ref first.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
make -s -j8 -C "$ROOT/oracle"
g++ -std=c++20 -O2 -I/root/reference/proj/include "$HERE/gen_golden.cpp" \
    "$ROOT/oracle/_ref/libmuxsim_core.a" -o "$ROOT/oracle/_ref/gen_golden"
"$ROOT/oracle/_ref/gen_golden" "$HERE"
g++ -std=c++20 -O2 -I/root/reference/proj/include "$HERE/gen_candidates.cpp" \
    "$ROOT/oracle/_ref/libmuxsim_core.a" -o "$ROOT/oracle/_ref/gen_candidates"
"$ROOT/oracle/_ref/gen_candidates" "$HERE"
