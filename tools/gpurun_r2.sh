timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r02_final_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r02_final_gpu_tests.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_final_gpu_tests.log
