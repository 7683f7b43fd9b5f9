timeout 2400 python bench.py --strong --layout cols > gpurun_out/r02_strong_cols_final.json 2> gpurun_out/r02_strong_cols_final.err; echo rc=$?
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r02_strong_cols_final.json') if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['e2e']['seconds'], d['time_to_tol']['seconds'], d['c5'] and d['c5'].get('value'), d['clocks'])"
