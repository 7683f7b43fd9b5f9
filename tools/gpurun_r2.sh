timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --strong --layout cols --steps 100 --warmup 3 --skip-e2e --no-c5-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cols world1', d['value'], d['time_to_tol'])"
timeout 900 python bench.py --strong --layout rows --steps 50 --warmup 3 --skip-e2e --skip-ttt --no-c5-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('rows world1', d['value'])"
