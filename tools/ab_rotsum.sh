for v in default ss2m3 ss2m4 ss8m1 ss4m3; do
  if [ $v = default ]; then unset BCN_LIB; else export BCN_LIB=build/variants/$v.so; fi
  ncu --nvtx --nvtx-include "head.fc1/" --metrics gpu__time_duration.sum --clock-control none -k regex:rotsum --csv --log-file gpurun_out/rs_$v.csv python tools/layer_times.py 128 > /dev/null 2>&1
  python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/rs_$v.csv')) if len(r)>5]
h=rows[0]; k=h.index('Kernel Name'); m=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]:
    d[r[k][:28]].append(float(r[m].replace(',','')))
print('$v', {a:(round(sum(b)/1e6,3),len(b)) for a,b in d.items()})
PY
done
