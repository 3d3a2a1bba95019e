#!/bin/bash
# build_variant.sh NAME "EXTRA nvcc flags": a variant of the library in paper_1210_4090_b200/build_NAME/
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -s -j8 -C "$ROOT/paper_1210_4090_b200" OBJDIR="$ROOT/paper_1210_4090_b200/build_$1" \
    LIB="$ROOT/paper_1210_4090_b200/build_$1/liblaxol_b200.so" EXTRA="$2" \
    "$ROOT/paper_1210_4090_b200/build_$1/liblaxol_b200.so" 2>&1 | grep -E "error" || true
ls "$ROOT/paper_1210_4090_b200/build_$1/liblaxol_b200.so"
