STEPS=1000 bash tools/lib_sweep.sh base cl1 base cl1 base cl1 2>&1
