for k in 1 2 3; do SWR_BUILD_K=$k python tools/march_scan.py 500 2000 2>&1 | sed "s/^/K=$k /"; done
