for v in "" envc1w5 envc1w6; do echo "== ${v:-product}"; PQLG_LIB_VARIANT=$v timeout 300 python tools/ab_actor.py 2>&1 | grep "N=16384 algo=0" | cut -c1-60; done
