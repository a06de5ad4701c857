out=gpurun_out
tag=${1:-x}
timeout 900 python tools/explore.py 16384 gauss 32 fb 2 >> $out/${tag}_explore.txt 2>&1
timeout 900 python tools/explore.py 4096 gauss 32 fb 30 >> $out/${tag}_explore.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:'k_' -c 40 --csv \
    --log-file $out/${tag}_w32.csv python tools/prof_run.py 16384 12 gauss 32 > /dev/null 2>&1
