#!/usr/bin/env python
"""Run a command; print its wall time and peak RSS (children) to stderr."""
import resource
import subprocess
import sys
import time

t0 = time.time()
rc = subprocess.call(sys.argv[1:])
ru = resource.getrusage(resource.RUSAGE_CHILDREN)
print(f"wall {time.time() - t0:.1f} s, peak RSS {ru.ru_maxrss / 1e6:.1f} GB, rc {rc}", file=sys.stderr)
sys.exit(rc)
