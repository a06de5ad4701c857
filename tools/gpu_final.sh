# Round-end evidence in one gpurun call: GPU tests, bench line, ncu launch
# lists + full captures (summarised on the box; the n=4096 report kept).
out=gpurun_out
tag=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > $out/${tag}_pytest.log 2>&1; echo "rc $?" >> $out/${tag}_pytest.log
timeout 1500 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
bash tools/gpu_ncu.sh $tag
python tools/ncu_summary.py $out/${tag}_launches_n4096.csv $out/${tag}_launches_n16384.csv $out/${tag}_full_n4096.ncu-rep \
    $out/${tag}_full_n16384.ncu-rep > $out/${tag}_ncu_summary.txt 2>&1
rm -f $out/${tag}_full_n16384.ncu-rep
