export PROF_G=64 PROF_LAYOUT=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:slot_major_ks -s 3 -c 1 -o gpurun_out/smks python tools/prof_kernels.py convks > gpurun_out/exp39_ncu.log 2>&1; echo rc=$?
