timeout 900 python -m pytest tests/test_gpu_primitives.py -x -q -m gpu -k "rotsum" 2>&1 | tail -2
python tools/prof_kernels.py rotsum3 > /dev/null && ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:"rotsum" -c 1 python tools/prof_kernels.py rotsum3 2>&1 | grep -E "duration|inst_exec"
python tools/g_sweep.py 128 2>&1 | grep "G="
