STEPS=1000 bash tools/lib_sweep.sh base prev base prev base prev 2>&1
