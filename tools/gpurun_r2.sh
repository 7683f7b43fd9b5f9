timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -x -q 2>&1 | tail -1
for i in 1 2 3; do
  STEPS=1000 bash tools/lib_sweep.sh base 2>&1
  CF_BENCH_NO_EVENTS=1 timeout 300 python bench.py --config c2 --steps 1000 --warmup 5 --skip-e2e --skip-cpu --skip-ttt 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['iteration_roofline']
print('noevents   it/s %7.1f  ms %.4f  clk %s' % (d['value'], r['ms_per_iteration'], d['clocks']['sm_mhz']))"
done
timeout 300 python bench.py --steps 20 --warmup 5 --skip-e2e --skip-cpu --skip-ttt 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline'], d['iteration_roofline'])"
