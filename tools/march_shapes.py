"""C5 build+final march times for forced launch shapes (SWR_MARCH_PMAX / SWR_MARCH_M)."""
import os, subprocess, sys
for env in ({}, {"SWR_MARCH_PMAX": "128", "SWR_MARCH_M": "11"}):
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "tools/quick_c5.py", "C5"], env=e, capture_output=True, text=True).stdout
    print(env, [l for l in out.splitlines() if l.startswith("status")][-1:])
