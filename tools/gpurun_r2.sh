timeout 900 python -m pytest tests -m gpu -q -x -k "batch or benchrun or checked" 2>&1 | tail -n 2
for l in old base; do
  if [ $l = base ]; then P=""; else P=paper_2203_05027_b200/libcfb200_$l.so; fi
  echo -n "$l one: "; CF_LIB_PATH=$P python tools/batch_one.py 2>&1 | tail -1
  CF_LIB_PATH=$P timeout 300 python bench.py --config c4 --skip-cpu --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$l', '%.1fM problem-it/s' % (d['value']/1e6), d['time_to_tol']['iters_total'], d['time_to_tol']['statuses'])"
done
