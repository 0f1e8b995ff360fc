mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prefill_launches.csv python tools/bench_prefill.py --bits 4 --iters 1 > gpurun_out/ncu_prefill.log 2>&1
tail -2 gpurun_out/ncu_prefill.log
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/prefill_launches.csv')))
h = rows[0]; ik = h.index('Kernel Name'); iv = h.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[2:]:
    if len(r) <= iv: continue
    try: v = float(r[iv].replace(',', ''))
    except ValueError: continue
    k = r[ik].split('(')[0][:60]
    agg[k][0] += 1; agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{t/1e3:9.1f} us {n:5d}x  {k}")
print("total", tot / 1e3, "us")
PY
