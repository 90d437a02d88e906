timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/time_ntt.py 32 2>&1 | tail -2
python tools/g_sweep.py 128 2>&1 | grep "G="
