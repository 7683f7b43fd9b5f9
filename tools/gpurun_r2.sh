set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_checked.py tests/test_gpu_variants.py -x -q 2>&1 | tail -4
STEPS=1000 bash tools/lib_sweep.sh base fd0 fu4 fu6 base fd0 2>&1
CFG=c3 STEPS=1000 bash tools/lib_sweep.sh base fd0 fu4 base fd0 2>&1
