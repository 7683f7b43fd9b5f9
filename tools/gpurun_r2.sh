CF_LIB_PATH=paper_2203_05027_b200/libcfb200_epf.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
STEPS=1000 bash tools/lib_sweep.sh base epf base epf base epf 2>&1
