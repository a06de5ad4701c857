# new GPU tests + racecheck variants + w=16 / w=32 sweep rates
out=gpurun_out
tag=${1:-r02i}
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 python -m pytest tests/test_gpu_accuracy.py tests/test_gpu_stripes.py tests/test_gpu_nccl.py \
    tests/test_gpu_parity.py tests/test_gpu_ops.py tests/test_gpu_northstar.py -q \
    --deselect tests/test_gpu_northstar.py::test_config4_illconditioned_dmma_vs_oracle \
    --deselect tests/test_gpu_northstar.py::test_config4_illconditioned_exact_bitwise_vs_oracle > $out/${tag}_pytest.log 2>&1
echo "rc $?" >> $out/${tag}_pytest.log
timeout 1200 $CS --tool racecheck --racecheck-report all --print-limit 20 --kernel-name-exclude kns=k_post \
    --log-file $out/${tag}_racecheck_nopost.log python tools/sanitize_run.py 256 > /dev/null 2>&1
timeout 1200 $CS --tool racecheck --racecheck-report analysis --print-limit 20 \
    --log-file $out/${tag}_racecheck_analysis.log python tools/sanitize_run.py 256 > /dev/null 2>&1
for w in 16 32; do
  timeout 600 python bench.py --steps 3 --warmup 3 --w $w --no-full --config4-size 0 --no-cpu > $out/${tag}_bench_w$w.json 2>&1
done
