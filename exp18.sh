timeout 900 python -m pytest tests/test_gpu_primitives.py -x -q -m gpu -k "conv_ks or planes" 2>&1 | tail -2
for gb in 16 32 8; do BCN_IMMA_GB=$gb timeout 300 python tools/time_ntt.py 32 2>&1 | tail -1; done
python tools/prof_kernels.py convks > /dev/null && ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:"mac_imma" -c 2 python tools/prof_kernels.py convks > gpurun_out/m.log 2>&1
grep -E "duration|tensor_cycles" gpurun_out/m.log
