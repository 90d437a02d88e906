# A/B of runtime switches on the cfg4 step (bench.py --no-extras), one box: default, BCN_SPLIT_CONV=0, BCN_FUSED_INNER=1, default
run() { python bench.py --steps 3 --warmup 3 --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"; }
run default
BCN_SPLIT_CONV=0 run split_conv0
BCN_FUSED_INNER=1 run fused_inner1
run default
