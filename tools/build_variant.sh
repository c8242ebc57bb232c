#!/bin/bash
# Build a tuning variant of libarfx.so with extra nvcc flags into lib/variants/NAME.so
# (own object dir; the default build is untouched). Usage: tools/build_variant.sh NAME "-DFOO=1 ..."
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2212_10550_b200/lib/variants
ARFX_NVCC_EXTRA="$2" ARFX_BUILD_DIR=build/var_$1 ARFX_LIB_OUT=paper_2212_10550_b200/lib/variants/$1.so \
  python -c "from paper_2212_10550_b200.build import build; build()"
