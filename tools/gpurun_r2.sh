CF_LIB_PATH=paper_2203_05027_b200/libcfb200_ee1.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
CF_LIB_PATH=paper_2203_05027_b200/libcfb200_ee2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
STEPS=1000 bash tools/lib_sweep.sh base ee1 ee2 base ee1 ee2 base ee1 ee2 2>&1
