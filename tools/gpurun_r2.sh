timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -x -q 2>&1 | tail -1
STEPS=1000 bash tools/lib_sweep.sh base prev base prev base prev 2>&1
