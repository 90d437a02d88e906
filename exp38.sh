export PROF_G=64 PROF_LAYOUT=1
for v in "-DUM_ST=3 -DUM_RS=2" "-DUM_ST=2 -DUM_RS=3" "-DUM_ST=2 -DUM_RS=2"; do
echo "== $v"; BCN_NVCC_EXTRA="-DBCN_UMMA_PROF $v" python -m paper_2402_01296_b200.build > /dev/null 2>&1 || echo BUILD_FAIL
timeout 300 python tools/prof_kernels.py convks 2>&1 | grep umma | tail -4
done
