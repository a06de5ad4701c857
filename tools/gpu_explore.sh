out=gpurun_out
python tools/phase_prof.py 4096 > $out/r01c_phase.txt 2>&1
for args in "4096 cond 16 fb 100" "4096 cond 16 bo 100" "4096 cond 32 fb 100" "4096 cond 32 bo 100" "4096 gauss 16 fb 30" "4096 gauss 32 fb 30" "16384 gauss 16 fb 2" "16384 gauss 32 fb 2" "16384 gauss 16 bo 2"; do
  set -- $args
  timeout 600 python tools/explore.py $1 $2 $3 $4 $5 >> $out/r01c_explore.txt 2>&1
done
