for d in 0 16; do echo "dbg=$d"; HX_TC_DEBUG=$d PROBE_REPS=3 python tools/mac_tc_probe.py 8 2>&1 | grep -o "'tc_ms_per_token': [0-9.]*"; done
