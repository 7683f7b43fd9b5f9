timeout 1200 python tools/e2e_sharded_profile.py 2>&1 | grep -v Warn | tail -4
