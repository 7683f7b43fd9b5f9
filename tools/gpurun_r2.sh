STEPS=1000 bash tools/lib_sweep.sh base cl base cl 2>&1
