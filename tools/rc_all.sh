out=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "repeatable or w32 or exact_mode_bitwise or fused" > $out/r02s2_pytest.log 2>&1; echo "rc $?" >> $out/r02s2_pytest.log
for w in 32 16; do timeout 400 python bench.py --steps 3 --warmup 3 --no-full --config4-size 0 --no-cpu --w $w > $out/r02s2_b$w.json 2>&1; python -c "import json; d=json.loads(open('$out/r02s2_b$w.json').read().strip().splitlines()[-1]); r=d['roofline']; print($w, round(d['value']), r['avg_launch_ms'], r['grammian']['avg_launch_ms'])" >> $out/r02s2.txt; done
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool racecheck --racecheck-report all --print-limit 10 --log-file $out/r02s2_racecheck.log python tools/sanitize_run.py 256 > $out/r02s2_racecheck.stdout 2>&1
grep SUMMARY $out/r02s2_racecheck.log >> $out/r02s2.txt
grep -o "at void hzg::<unnamed>::[a-z_]*<[^>]*>" $out/r02s2_racecheck.log | sort | uniq -c >> $out/r02s2.txt
