out=gpurun_out
tag=${1:-r02u}
run() {
  env "$@" timeout 400 python bench.py --steps 3 --warmup 3 --no-full --config4-size 0 --no-cpu > $out/${tag}_tmp.json 2>&1
  python -c "import json,sys; d=json.loads(open('$out/${tag}_tmp.json').read().strip().splitlines()[-1]); print('$*', round(d['value']), round(d['s_per_sweep'],4), d['clocks']['sm_mhz'], d['roofline']['inner']['avg_launch_ms'])" >> $out/${tag}_tune.txt 2>&1
}
run HZG_INNER_SMEM=0
run HZG_INNER_SMEM=116
run HZG_INNER_SMEM=116 HZG_DEFER_Z=0
run HZG_INNER_SMEM=120 HZG_GROUPS=16
run HZG_INNER_SMEM=0 HZG_GROUPS=16
