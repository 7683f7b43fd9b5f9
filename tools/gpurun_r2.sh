timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r02_final_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r02_final_gpu_tests.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_final_gpu_tests.log
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/final_$name.json 2> gpurun_out/final_$name.err; echo "$name rc=$?"; }
run c2
run ref_c2 --impl reference
run c4 --config c4
