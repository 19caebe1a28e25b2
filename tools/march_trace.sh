# per-CTA phase trace + build-march timing of C5 (rebuilds libswr.so with the
# trace points compiled in; SWR_TRACE=1 adds one traced launch per march)
SWR_TRACE_BUILD=1 python paper_1503_02564_b200/_build.py > /dev/null || exit 1
SWR_TRACE_BUILD=1 SWR_TRACE=1 timeout 120 python tools/march_scan.py 500 2>&1
python paper_1503_02564_b200/_build.py > /dev/null
