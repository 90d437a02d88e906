export PROF_G=64 PROF_LAYOUT=1
for d in 0 16; do echo "dbg=$d"; BCN_UMMA_DBG=$d timeout 300 python tools/prof_kernels.py convks 2>&1 | grep umma | tail -4; done
