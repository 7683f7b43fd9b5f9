# launch list of the bench command (cold-cache serialised times: the share of the step is what counts)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches.csv python bench.py --steps 20 --warmup 5 --warm-seconds 0 --skip-e2e --skip-ttt --skip-cpu > gpurun_out/r02b_launch_bench.log 2>&1
echo launch rc=$?
# one full capture of the passes (row panel 1, row panel 2, column pass) of the bench iteration
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"RowIter|ColIter" -c 3 -o gpurun_out/r02b_c2_full -f python tools/prof_iter.py --config c2 --iters 2 > gpurun_out/r02b_full.log 2>&1
echo full rc=$?
