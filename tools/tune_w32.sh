# sweep-rate tuning at config 5 (w=32): position groups, deferred Z, priorities
out=gpurun_out
tag=${1:-r02p}
run() {
  env "$@" timeout 400 python bench.py --steps 3 --warmup 3 --no-full --config4-size 0 --no-cpu > $out/${tag}_tmp.json 2>&1
  python -c "import json,sys; d=json.loads(open('$out/${tag}_tmp.json').read().strip().splitlines()[-1]); print('$*', round(d['value']), round(d['s_per_sweep'],4), d['clocks']['sm_mhz'])" >> $out/${tag}_tune.txt 2>&1
}
run HZG_GROUPS=8
run HZG_GROUPS=4
run HZG_GROUPS=16
run HZG_GROUPS=2
run HZG_DEFER_Z=0
run HZG_PRIO=0
run HZG_INNER_PRIO=1
run HZG_GROUPS=8
run HZG_INNER_CTAS=16
run HZG_INNER_CTAS=24
