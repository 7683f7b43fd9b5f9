for lib in base nc1 nc2 base; do
  if [ "$lib" = base ]; then path=""; else path="paper_2203_05027_b200/libcfb200_$lib.so"; fi
  echo -n "$lib: "; CF_LIB_PATH=$path timeout 120 python tools/cluster_one.py 2>&1 | tail -1
done
