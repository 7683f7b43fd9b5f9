for c in c1 c3 c3m c4; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 5 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "$c rc=$?"
done
for c in c1 c3 c4; do
  timeout 900 python bench.py --config $c --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_reference_$c.json 2> gpurun_out/r02_bench_reference_$c.err; echo "ref $c rc=$?"
done
timeout 900 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/r02_bench_c5_full_scale_1gpu.json 2> gpurun_out/r02_bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --config c5 --c5-mode cols --steps 20 --warmup 3 > gpurun_out/r02_bench_c5_cols_1gpu.json 2> gpurun_out/r02_bench_c5c.err; echo "c5 cols rc=$?"
