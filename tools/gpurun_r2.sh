timeout 600 python tools/loop_overhead.py c2 2>&1 | tail -8
