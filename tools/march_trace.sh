# per-CTA phase trace + build-march timing of C5 (SWR_TRACE=1 adds one traced launch per march)
SWR_TRACE=1 python tools/march_scan.py 500 2>&1
