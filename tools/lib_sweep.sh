#!/bin/bash
# usage: tools/lib_sweep.sh [config] lib1 lib2 ...   (lib "base" = the product build)
# one short bench per library build, interleaved; prints it/s, per-pass ms and the clock
cfg=${CFG:-c2}
for lib in "$@"; do
  if [ "$lib" = base ]; then path=""; else path="paper_2203_05027_b200/libcfb200_$lib.so"; fi
  CF_LIB_PATH=$path timeout 300 python bench.py --config $cfg --steps ${STEPS:-500} --warmup 5 --skip-e2e --skip-cpu --skip-ttt 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['iteration_roofline']
print('%-10s it/s %7.1f  ms %.4f  row %.4f  col %.4f  frac %.3f  clk %s' % ('$lib', d['value'], r['ms_per_iteration'], r['row_pass_ms'], r['col_pass_ms'], r['frac'], d['clocks']['sm_mhz']))"
done
