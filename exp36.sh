export PROF_G=64 PROF_LAYOUT=1
for d in 0 1 2 4 3 7; do
BCN_UMMA_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp36_$d.csv python tools/prof_kernels.py convks > /dev/null 2>&1; echo rc=$?
done
