out=gpurun_out
tag=${1:-x}
timeout 600 python -m pytest tests -m gpu -x -q > $out/${tag}_pytest.log 2>&1; echo "rc $?" >> $out/${tag}_pytest.log
python tools/phase_prof.py 4096 >> $out/${tag}_phase.txt 2>&1
timeout 1200 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
