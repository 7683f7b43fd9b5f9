timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_checked.py tests/test_gpu_sharded.py tests/test_gpu_variants.py -x -q 2>&1 | tail -2
STEPS=1000 bash tools/lib_sweep.sh base prev base prev 2>&1
CFG=c3 STEPS=1000 bash tools/lib_sweep.sh base prev base prev 2>&1
