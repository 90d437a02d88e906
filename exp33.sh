export PROF_G=64 PROF_LAYOUT=1
timeout 300 python tools/prof_kernels.py convks && echo OK_PLAIN
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp33_launch.csv python tools/prof_kernels.py convks > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mac_umma -s 1 -c 1 -o gpurun_out/umma python tools/prof_kernels.py convks > gpurun_out/exp33_ncu.log 2>&1; echo rc=$?
