#!/bin/bash
# A/B variant of libpqlg.so: same sources, extra nvcc flags, loaded with
# PQLG_LIB_VARIANT=<name>.   tools/build_variant.sh <name> "-DFOO=1 ..."
cd "$(dirname "$0")/.." && PQLG_VARIANT_NAME="$1" PQLG_NVCC_EXTRA="$2" python paper_2307_12983_b200/build.py
