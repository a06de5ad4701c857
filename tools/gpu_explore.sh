out=gpurun_out
tag=${1:-x}
for g in 1 2 4 8 16; do
  echo "groups $g" >> $out/${tag}_explore.txt
  HZG_GROUPS=$g timeout 900 python tools/explore.py 16384 gauss 16 fb 2 >> $out/${tag}_explore.txt 2>&1
done
