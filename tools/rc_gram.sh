out=gpurun_out
for w in 32 16; do timeout 400 python bench.py --steps 3 --warmup 3 --no-full --config4-size 0 --no-cpu --w $w > $out/r02r2_b$w.json 2>&1; python -c "import json; d=json.loads(open('$out/r02r2_b$w.json').read().strip().splitlines()[-1]); r=d['roofline']; print($w, round(d['value']), r['grammian']['avg_launch_ms'])" >> $out/r02r2.txt; done
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool racecheck --racecheck-report all --print-limit 10 --kernel-name-exclude kns=k_post --log-file $out/r02r2_racecheck_nopost.log python tools/sanitize_run.py 256 > /dev/null 2>&1
grep SUMMARY $out/r02r2_racecheck_nopost.log >> $out/r02r2.txt
