out=gpurun_out
tag=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > $out/${tag}_pytest.log 2>&1; echo "rc $?" >> $out/${tag}_pytest.log
python tools/phase_prof.py 4096 > $out/${tag}_phase.txt 2>&1
timeout 600 python tools/explore.py 4096 cond 16 fb 100 >> $out/${tag}_explore.txt 2>&1
