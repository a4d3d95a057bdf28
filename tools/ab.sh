# A/B helper for gpurun: launch list of two frames + the default bench line
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/ll.csv python tools/profile_step.py --frames 2 --warmup 2 > gpurun_out/ll.log 2>&1
timeout 300 python bench.py "$@" > gpurun_out/b4.log 2>&1
python - <<'PY'
import csv, json
l = [x for x in open('gpurun_out/b4.log') if x.startswith('{')][-1]
d = json.loads(l)
print(d['value'], d['e2e']['value'], d['roofline']['stages_ms'])
rows = list(csv.reader(open('gpurun_out/ll.csv')))
h = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[h]; ii = hdr.index('ID'); ki = hdr.index('Kernel Name'); mi = hdr.index('Metric Name'); vi = hdr.index('Metric Value')
ks = {}
for r in rows[h + 1:]:
    if len(r) > vi:
        ks.setdefault(r[ii], [r[ki][:48], 0.0, 0.0])
        ks[r[ii]][1 if r[mi].startswith('gpu__time') else 2] = float(r[vi].replace(',', ''))
for name, t, n in list(ks.values())[-13:]:
    print(f"{t / 1000:8.1f} us {n / 1e6:8.2f} M  {name}")
PY
