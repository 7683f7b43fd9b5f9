mkdir -p gpurun_out
for cfg in "48 48" "40 48" "32 48" "28 48" "24 48" "64 48" "48 24" "48 32" "32 24"; do
  set -- $cfg
  echo "PANEL=$1 BAND=$2" >> gpurun_out/sweep.log
  CF_PANEL_MB=$1 CF_BAND_MB=$2 timeout 300 python tools/prof_iter.py --config c2 --iters 400 >> gpurun_out/sweep.log 2>&1
done
for cfg in "48 48" "32 48" "24 48" "48 24"; do
  set -- $cfg
  echo "C3 PANEL=$1 BAND=$2" >> gpurun_out/sweep.log
  CF_PANEL_MB=$1 CF_BAND_MB=$2 timeout 300 python tools/prof_iter.py --config c3 --iters 400 >> gpurun_out/sweep.log 2>&1
done
