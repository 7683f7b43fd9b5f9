for l in s512m2 s512m3; do for c in plan plan_knobs; do CF_LIB_PATH=paper_2203_05027_b200/libcfb200_$l.so timeout 300 python tools/sanitize_cases.py $c 2>&1 | tail -1; done; done
bash tools/lib_sweep.sh base s512m2 s512m3 base s512m2 s512m3
CFG=c3 bash tools/lib_sweep.sh base s512m2 s512m3
