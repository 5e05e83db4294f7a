# per-kernel durations of the headline step for two builds (MCF_LIB), last step only
for L in old b200; do
MCF_LIB=$PWD/paper_2207_08867_b200/libmcf_$L.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_$L.csv python tools/headline_steps.py > /dev/null 2>&1
python - <<PY
import csv,collections
rows=[r for r in csv.reader(open("gpurun_out/ab_$L.csv")) if len(r)>5]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
d=collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki][:40]].append(float(r[vi].replace(",","")))
print("$L", {k:round(sum(v[-max(1,len(v)//5):])/1000,2) for k,v in d.items()})
PY
done
