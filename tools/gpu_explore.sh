out=gpurun_out
tag=${1:-x}
for pc in 1024 512 256; do for sr in 0 256; do
  echo "post chunk $pc split rows $sr" >> $out/${tag}_explore.txt
  if [ $sr = 0 ]; then HZG_POST_CHUNK=$pc timeout 900 python tools/explore.py 4096 cond 16 fb 100 >> $out/${tag}_explore.txt 2>&1;
  else HZG_SPLIT_ROWS=$sr HZG_POST_CHUNK=$pc timeout 900 python tools/explore.py 4096 cond 16 fb 100 >> $out/${tag}_explore.txt 2>&1; fi
done; done
