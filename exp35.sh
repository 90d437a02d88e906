export PROF_G=64 PROF_LAYOUT=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mac_umma -s 2 -c 1 -o gpurun_out/umma2 python tools/prof_kernels.py convks > gpurun_out/exp35_ncu.log 2>&1; echo rc=$?
