bash tools/lib_sweep.sh base h1 h2 x1 h1x1 h2x2 base h1 h2 x1 h1x1 h2x2
