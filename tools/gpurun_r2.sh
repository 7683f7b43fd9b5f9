timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/r2_t2_all.log 2>&1; echo "all rc=$?"
tail -n 12 gpurun_out/r2_t2_all.log
