timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sc_launch.csv python scripts/scatter_prof.py > /dev/null 2>&1
python - <<'P'
import csv
rows=[r for r in csv.DictReader([l for l in open('gpurun_out/sc_launch.csv') if l.startswith('"')])]
cur=None
for r in rows:
    k=(r['ID'], r['Kernel Name'][:50])
    if k!=cur:
        cur=k; print()
        print(r['ID'], r['Kernel Name'][:50], end=' ')
    print(r['Metric Name'].split('.')[0][-14:], r['Metric Value'], r['Metric Unit'], end=' | ')
print()
P
