# Round-2 evidence in one gpurun call: GPU tests, the bench line (default:
# config 5 at w=32 + full solve + config 4 + CPU sample), the reference arm,
# ncu launch lists and full captures (w=32 n=16384 bench workload, w=16
# n=4096 config 4), summarised on the box.
out=gpurun_out
tag=${1:-r02z}
timeout 2400 python -m pytest tests -m gpu -q > $out/${tag}_pytest.log 2>&1; echo "rc $?" >> $out/${tag}_pytest.log
timeout 1500 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
timeout 900 python bench.py --impl reference > $out/${tag}_bench_ref.json 2> $out/${tag}_bench_ref.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:'k_' -c 60 --csv \
    --log-file $out/${tag}_launches_w32_n16384.csv python tools/prof_run.py 16384 12 gauss 32 > $out/${tag}_l1.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:'k_' -c 2000 --csv \
    --log-file $out/${tag}_launches_w16_n4096.csv python tools/prof_run.py 4096 255 cond 16 > $out/${tag}_l2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_post|k_gram|k_inner' -s 6 -c 3 \
    -o $out/${tag}_full_w32_n16384 -f python tools/prof_run.py 16384 4 gauss 32 > $out/${tag}_f1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_post|k_gram|k_inner' -s 30 -c 3 \
    -o $out/${tag}_full_w16_n4096 -f python tools/prof_run.py 4096 20 cond 16 > $out/${tag}_f2.log 2>&1
python tools/ncu_summary.py $out/${tag}_launches_w32_n16384.csv $out/${tag}_launches_w16_n4096.csv \
    $out/${tag}_full_w32_n16384.ncu-rep $out/${tag}_full_w16_n4096.ncu-rep > $out/${tag}_ncu_summary.txt 2>&1
python tools/ncu_traffic.py $out/${tag}_full_w32_n16384.ncu-rep $out/${tag}_traffic_w32_n16384.json > /dev/null 2>&1
# the captures stay on the box (gpurun copies back <= 64 MiB): keep the
# summaries and a source-level table of the inner kernel at n = 4096
ncu -i $out/${tag}_full_w16_n4096.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_inner \
    > $out/${tag}_inner_source_w16_n4096.csv 2>/dev/null
gzip -f $out/${tag}_inner_source_w16_n4096.csv
rm -f $out/*.ncu-rep
du -sh $out
