timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_t7_all.log 2>&1; echo "all rc=$?"
tail -n 1 gpurun_out/r2_t7_all.log
bash tools/lib_sweep.sh old base nocarve old base nocarve
CFG=c3 bash tools/lib_sweep.sh old base nocarve
CFG=c3m bash tools/lib_sweep.sh old base nocarve
for l in old base; do
  if [ $l = base ]; then P=""; else P=paper_2203_05027_b200/libcfb200_$l.so; fi
  echo "== $l"; CF_LIB_PATH=$P timeout 600 python tools/prof_sizes.py 2>&1 | tail -7
done
