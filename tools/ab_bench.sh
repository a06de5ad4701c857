# A/B of bench.py under env settings: prints value, ms/step, SM clock per setting
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$cfg', round(d['value']), round(d['ms_per_step']), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],2))"
done
