# A/B of libbcn build variants (build/variants/<name>.so, loaded through BCN_LIB) on one box:
# config 3 (tools/time_cfg3.py) and the cfg4 step (bench.py --no-extras).  usage: bash tools/ab_lib.sh default v1 v2 ...
for v in "$@"; do
  if [ $v = default ]; then unset BCN_LIB; else export BCN_LIB=$PWD/build/variants/$v.so; fi
  echo "== $v"
  python tools/time_cfg3.py 2>&1 | tail -1
  python bench.py --steps 3 --warmup 3 --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', round(d['value']), 'images/s', round(d['ms_per_step'],1), 'ms', d['clocks']['sm_mhz'])"
done
