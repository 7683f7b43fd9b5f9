timeout 1200 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; echo rc=$?
python -c "
import json; d=json.loads([l for l in open('gpurun_out/final_c2.json') if l.startswith('{')][-1]); print(d['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['passes'], d['clocks'], d['cpu_baseline']['value'], d['e2e']['value'])"
