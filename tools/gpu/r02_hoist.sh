for hc in 8 16 32; do HOIST_CHUNK=$hc HX_TAG=chunk$hc timeout 600 python tools/ks_time.py 256 hoisted 2>&1 | tail -1; done
