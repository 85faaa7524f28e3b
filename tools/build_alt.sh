#!/usr/bin/env bash
# Build an A/B variant of libspa2.so with extra compile-time flags into alt/<name>/libspa2.so
# (git-ignored, ships to the GPU box); time it with `python bench.py --lib alt/<name>/libspa2.so`.
#   bash tools/build_alt.sh nk4 -DSPA2_DQ_NK=4
set -eu
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
D="$ROOT/alt/$NAME"
rm -rf "$D"; mkdir -p "$D/pkg/csrc" "$D/include"
cp "$ROOT"/paper_2602_13515_b200/csrc/*.cu "$ROOT"/paper_2602_13515_b200/csrc/*.cuh "$ROOT"/paper_2602_13515_b200/csrc/*.h \
   "$ROOT"/paper_2602_13515_b200/csrc/Makefile "$D/pkg/csrc/" 2>/dev/null || true
cp "$ROOT"/include/spa2.h "$ROOT"/include/spa2_diag.h "$D/include/"
make -s -C "$D/pkg/csrc" -j 8 EXTRA_NVFLAGS="$*" ../libspa2.so >/dev/null
mv "$D/pkg/libspa2.so" "$D/libspa2.so"
rm -rf "$D/pkg" "$D/include"
echo "$D/libspa2.so"
