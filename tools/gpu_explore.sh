out=gpurun_out
tag=${1:-x}
HZG_SPLIT_ROWS=256 timeout 900 python -m pytest tests -m gpu -x -q -k "fused" > $out/${tag}_pytest_fused.log 2>&1; echo "rc $?" >> $out/${tag}_pytest_fused.log
echo "fused split 256" >> $out/${tag}_explore.txt
HZG_SPLIT_ROWS=256 timeout 900 python tools/explore.py 16384 gauss 16 fb 2 >> $out/${tag}_explore.txt 2>&1
echo "unfused split 256" >> $out/${tag}_explore.txt
HZG_SPLIT_ROWS=256 HZG_FUSED=0 timeout 900 python tools/explore.py 16384 gauss 16 fb 2 >> $out/${tag}_explore.txt 2>&1
echo "unfused split 512" >> $out/${tag}_explore.txt
HZG_FUSED=0 timeout 900 python tools/explore.py 16384 gauss 16 fb 2 >> $out/${tag}_explore.txt 2>&1
