# ncu evidence for the step kernels (one GPU): launch list of one full
# sweep-1 pass at n=4096 and full captures of the three step kernels.
out=gpurun_out
tag=${1:-x}
n=${2:-4096}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_|k_' -c 2000 --csv \
    --log-file $out/${tag}_launches.csv python tools/prof_run.py $n 255 cond > $out/${tag}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_post|k_gram|k_inner' -s 30 -c 3 \
    -o $out/${tag}_full -f python tools/prof_run.py $n 20 cond > $out/${tag}_full.log 2>&1
