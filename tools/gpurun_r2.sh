mkdir -p gpurun_out/san
nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.sw_power_cap,power.draw --format=csv,noheader -lms 200 > gpurun_out/ideal_clocks.csv &
SMI=$!
timeout 300 ./scratch/ideal_iter_probe 2000 > gpurun_out/r2_ideal_iter_probe.txt 2>&1; echo "ideal rc=$?"
kill $SMI
cat gpurun_out/r2_ideal_iter_probe.txt
sort gpurun_out/ideal_clocks.csv | uniq -c | sort -rn | head -5
for tool in memcheck racecheck synccheck; do
  for case in plan plan_knobs cluster1 cluster8 cluster16 batch gen; do
    timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python tools/sanitize_cases.py $case > gpurun_out/san/${tool}_${case}.log 2>&1
    echo "$tool $case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${tool}_${case}.log | tail -1) $(grep -c 'case .*: ok' gpurun_out/san/${tool}_${case}.log)"
  done
done
