out=gpurun_out
tag=${1:-x}
python tools/phase_prof.py 4096 > $out/${tag}_phase.txt 2>&1
HZG_LIB=scratch/nomath/libhzg_nomath.so python tools/phase_prof.py 4096 >> $out/${tag}_phase.txt 2>&1
timeout 900 python tools/cmp_cond1024.py > $out/${tag}_cmp1024.txt 2>&1
