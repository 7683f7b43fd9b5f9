run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/final_$name.json 2> gpurun_out/final_$name.err; echo "$name rc=$?"; }
run c2
run c3 --config c3
run c3m --config c3m
