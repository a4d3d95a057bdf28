# A/B helper for gpurun: launch list of two frames + the default bench line
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll.csv python tools/profile_step.py --frames 2 --warmup 2 > gpurun_out/ll.log 2>&1
timeout 300 python bench.py "$@" > gpurun_out/b4.log 2>&1
python - <<'PY'
import csv, json
l = [x for x in open('gpurun_out/b4.log') if x.startswith('{')][-1]
d = json.loads(l)
print(d['value'], d['e2e']['value'], d['roofline']['stages_ms'])
rows = list(csv.reader(open('gpurun_out/ll.csv')))
h = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[h]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
ks = [(r[ki][:48], float(r[vi].replace(',', ''))) for r in rows[h + 1:] if len(r) > vi]
for k, v in ks[-13:]:
    print(f"{v / 1000:8.1f} us  {k}")
PY
