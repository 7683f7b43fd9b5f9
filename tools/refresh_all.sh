# Re-measure every bench config on the current build (one box, one sitting); lines land in gpurun_out/final_*.json
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/final_$name.json 2> gpurun_out/final_$name.err; echo "$name rc=$?"; }
run c1 --config c1
run c3 --config c3
run c3m --config c3m
run c4 --config c4
run c5 --config c5 --c5-scale 0.1
run c5_p2p --config c5 --c5-scale 0.1 --c5-mode p2p
run c5_auto --config c5 --c5-scale 0.1 --c5-mode auto
run ref_c1 --impl reference --config c1
run ref_c3 --impl reference --config c3
run ref_c4 --impl reference --config c4
