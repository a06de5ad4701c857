out=gpurun_out
tag=${1:-x}
for g in 4 8 16 32 64; do
  echo "groups $g" >> $out/${tag}_explore.txt
  HZG_GROUPS=$g timeout 600 python tools/explore.py 4096 cond 16 fb 100 >> $out/${tag}_explore.txt 2>&1
done
./tools/lat_bench >> $out/${tag}_lat.txt 2>&1
timeout 900 python tools/explore.py 16384 gauss 16 fb 30 >> $out/${tag}_explore.txt 2>&1
