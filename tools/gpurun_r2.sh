for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_profiling.py -x -q 2>&1 | grep -E "passed|failed|assert|Error" | head -3; done
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; echo "c2 rc=$?"
