#!/bin/bash
# A/B of bench_configs (CONFIGS, e.g. "4") for LIBS, 2 alternating rounds
for i in 1 2; do for L in $LIBS; do
  PMH_LIB_PATH=$PWD/$L timeout 600 python tools/bench_configs.py --configs ${CONFIGS:-4} 2>/dev/null | python -c "
import json,sys
out=[]
for l in sys.stdin:
    try: d=json.loads(l); out.append((d.get('algo'), round(d['ms_min'],2), d.get('sig_checksum',0) % 100000))
    except Exception: pass
print('$L'.split('/')[-1], out)
"; done; done
