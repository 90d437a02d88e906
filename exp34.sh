timeout 300 python -m pytest tests/test_gpu_primitives.py -x -q -m gpu -k "conv_ks" 2>&1 | tail -3
export PROF_G=64 PROF_LAYOUT=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp34_launch.csv python tools/prof_kernels.py convks > /dev/null 2>&1; echo rc=$?
unset PROF_G PROF_LAYOUT
timeout 300 python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/exp34_bench.json 2> gpurun_out/exp34_bench.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/exp34_bench.json'));print(d['value'],d['ms_per_step'])"
