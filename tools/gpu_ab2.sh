#!/bin/bash
# A/B of library variants (tools/build_variant.sh) on the update / actor step
mkdir -p gpurun_out
for v in "" $VARIANTS; do
  echo "== variant '${v:-product}'"
  PQLG_LIB_VARIANT=$v timeout 300 python tools/ab_update.py 2>&1 | tail -1
  PQLG_LIB_VARIANT=$v timeout 300 python tools/ab_actor.py 2>&1 | grep "N=16384 algo=0"
done
exit 0
