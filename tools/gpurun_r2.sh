timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_checked.py -x -q 2>&1 | tail -2
for lib in base prev base prev; do
  if [ "$lib" = base ]; then path=""; else path="paper_2203_05027_b200/libcfb200_$lib.so"; fi
  echo -n "$lib: "; CF_LIB_PATH=$path timeout 120 python tools/cluster_one.py 2>&1 | tail -1
done
python tools/cluster_sizes.py 2>&1 | tail -12
