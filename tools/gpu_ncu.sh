# ncu evidence for the step kernels (one GPU): launch list of sweep 1 at
# n=4096 (config 4) and n=16384 (iid Gaussian, 12 steps), full captures of
# the three step kernels at both sizes.
out=gpurun_out
tag=${1:-x}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_' -c 2000 --csv \
    --log-file $out/${tag}_launches_n4096.csv python tools/prof_run.py 4096 255 cond > $out/${tag}_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_' -c 40 --csv \
    --log-file $out/${tag}_launches_n16384.csv python tools/prof_run.py 16384 12 gauss > $out/${tag}_launches2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_post|k_gram|k_inner' -s 30 -c 3 \
    -o $out/${tag}_full_n4096 -f python tools/prof_run.py 4096 20 cond > $out/${tag}_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_post|k_gram|k_inner" -s 6 -c 3 \
    -o $out/${tag}_full_n16384 -f python tools/prof_run.py 16384 4 gauss > $out/${tag}_full2.log 2>&1
