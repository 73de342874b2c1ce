for c in 2 4 8 16; do HX_PIPE_CHUNK=$c timeout 300 python tools/e2e_timing.py 2>&1 | grep -E "chunk|duplex|h2d|d2h" | tr '\n' ' '; echo; done
