O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02q_launches.csv python tools/one_build.py C5 2 > $O/r02q.log 2>&1
python - <<'PY' > gpurun_out/r02q_list.txt
import csv, io
txt=open('gpurun_out/r02q_launches.csv').read()
txt=txt[txt.index('"ID"'):]
rows=[r for r in csv.DictReader(io.StringIO(txt)) if r.get("Metric Name")=="gpu__time_duration.sum"]
half=len(rows)//2
for r in rows[half:]:
    v=float(r["Metric Value"]); u=r["Metric Unit"]
    v = v/1e3 if u in ("nsecond","ns") else (v*1e3 if u in ("msecond","ms") else v)
    print("%10.1f us  %s  grid=%s block=%s" % (v, r["Kernel Name"][:90], r.get("Grid Size"), r.get("Block Size")))
PY
rm -f $O/r02q_launches.csv
cat $O/r02q_list.txt | sort -rn | head -40; wc -l $O/r02q_list.txt
