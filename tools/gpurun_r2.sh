timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py tests/test_gpu_headline.py -x -q 2>&1 | tail -n 2
bash tools/lib_sweep.sh old base def5 def4 bar5 old base def5 def4 bar5
CFG=c3 bash tools/lib_sweep.sh old base def5 def4 bar5
