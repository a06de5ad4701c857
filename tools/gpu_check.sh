#!/bin/bash
# One gpurun call: GPU tests, bench line, ncu launch list and full captures.
# Usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tag]
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/${tag}_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc $?" >> $out/${tag}_pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > $out/${tag}_bench.json 2> $out/${tag}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $out/${tag}_launches.csv \
    python tools/prof_run.py 4096 8 cond > $out/${tag}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_post|k_gram|k_inner' -s 6 -c 3 \
    -o $out/${tag}_prof -f python tools/prof_run.py 4096 4 cond > $out/${tag}_ncu_full.log 2>&1
