timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/prof_count.py --iters 3 --pv 1 2>&1 | tail -1 | cut -c1-80
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l_pv.csv python tools/prof_count.py --iters 1 --pv 1 > /dev/null 2>&1
python - <<'PY'
import csv,io
txt=open('gpurun_out/l_pv.csv').read()
rows=list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
for r in rows:
    n=r['Kernel Name']
    if 'k_join' in n or 'k_pv_rows' in n:
        print(n[:30], r['Metric Name'], r['Metric Value'])
PY
