timeout 900 python -m pytest tests/test_rls.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
CFG=c3m STEPS=1000 bash tools/lib_sweep.sh base checked 2>&1 | head -1
CF_NO_COL_RUNS=1 CFG=c3m STEPS=1000 bash tools/lib_sweep.sh base 2>&1
CFG=c3m STEPS=1000 bash tools/lib_sweep.sh base 2>&1
CF_NO_COL_RUNS=1 CFG=c3m STEPS=1000 bash tools/lib_sweep.sh base 2>&1
