# per-kernel durations (ncu, one pass) of the conv2-shape staging + MAC for the default build and BCN_LIB variants
export PROF_LVL=8 PROF_OUT=8 PROF_ROTS=16 PROF_REPS=0
for v in "$@"; do
  if [ $v = default ]; then unset BCN_LIB; else export BCN_LIB=build/variants/$v.so; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"slot_major_ks|mac_umma" -s 6 -c 12 --csv --log-file gpurun_out/ab_$v.csv python tools/time_convks.py > /dev/null 2>&1
  python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/ab_$v.csv')) if len(r)>5]
h=rows[0]; k=h.index('Kernel Name'); m=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]:
    d[r[k][:28]].append(float(r[m].replace(',','')))
print('$v', {a:round(sum(b)/len(b)/1e6,4) for a,b in d.items()})
PY
done
