timeout 900 python -m pytest tests/test_gpu_primitives.py -x -q -m gpu -k "conv_ks" 2>&1 | tail -3
