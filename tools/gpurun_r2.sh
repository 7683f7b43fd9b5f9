timeout 900 python bench.py --strong --layout cols --steps 50 --warmup 3 --c5-scale 0.1 > gpurun_out/r02_strong_cols.json 2> gpurun_out/r02_strong_cols.err; echo "cols rc=$?"
timeout 900 python bench.py --strong --layout rows --steps 50 --warmup 3 --no-c5-extra > gpurun_out/r02_strong_rows.json 2> gpurun_out/r02_strong_rows.err; echo "rows rc=$?"
tail -n 3 gpurun_out/r02_strong_cols.err gpurun_out/r02_strong_rows.err
cat gpurun_out/r02_strong_cols.json gpurun_out/r02_strong_rows.json
