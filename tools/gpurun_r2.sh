CF_LIB_PATH=paper_2203_05027_b200/libcfb200_ed.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -x -q 2>&1 | tail -2
STEPS=1000 bash tools/lib_sweep.sh base ed base ed 2>&1
CFG=c3 STEPS=1000 bash tools/lib_sweep.sh base ed 2>&1
