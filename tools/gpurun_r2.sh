nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap --format=csv -lms 500 > gpurun_out/r02_clocks.csv &
SMI=$!
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref_c2.json 2> gpurun_out/r02_bench_ref_c2.err; echo "ref rc=$?"
kill $SMI
CMD="python bench.py --steps 20 --warmup 5 --warm-seconds 0 --skip-e2e --skip-cpu --skip-ttt"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_pass|k_row_report|k_finalize|k_col|k_big" -c 200 --csv --log-file gpurun_out/r02_c2_launches.csv $CMD > /dev/null 2>&1; echo "launches rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_pass" -s 6 -c 3 -o gpurun_out/r02_c2_prof $CMD > gpurun_out/r02_ncu_full.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/ | tail -5
