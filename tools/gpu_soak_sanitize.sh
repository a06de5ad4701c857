out=gpurun_out
tag=${1:-r02g}
timeout 1500 python tools/soak.py 400 7 > $out/${tag}_soak.txt 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --print-limit 20 --log-file $out/${tag}_memcheck.log python tools/sanitize_run.py 256 > $out/${tag}_memcheck.stdout 2>&1
timeout 1500 $CS --tool synccheck --print-limit 20 --log-file $out/${tag}_synccheck.log python tools/sanitize_run.py 256 > $out/${tag}_synccheck.stdout 2>&1
timeout 1500 $CS --tool racecheck --racecheck-report all --print-limit 20 --kernel-name-exclude kns=k_post \
    --log-file $out/${tag}_racecheck_nopost.log python tools/sanitize_run.py 256 > $out/${tag}_racecheck.stdout 2>&1
