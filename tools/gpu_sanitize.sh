# compute-sanitizer evidence for the step kernels (one GPU): racecheck and
# synccheck (shared memory hazards, barrier misuse) and memcheck on small
# solves (tools/sanitize_run.py); logs land in gpurun_out/.
out=gpurun_out
tag=${1:-r02}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --log-file $out/${tag}_sanitize_${tool}.log \
      python tools/sanitize_run.py 256 > $out/${tag}_sanitize_${tool}.stdout 2>&1
  echo "$tool rc $?" >> $out/${tag}_sanitize_rc.txt
done
