timeout 600 python -m pytest tests/test_gpu_profiling.py -x -q 2>&1 | tail -3
