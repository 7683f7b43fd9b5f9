for lib in base s4 s2 m5 t128 base s4 s2 m5 t128; do
  if [ "$lib" = base ]; then path=""; else path="paper_2203_05027_b200/libcfb200_$lib.so"; fi
  CF_LIB_PATH=$path timeout 300 python bench.py --config c4 --skip-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', '%.1f M problem-it/s' % (d['value']/1e6))"
done
