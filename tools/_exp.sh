python tools/sweep_time.py 16384 3 4 32 0 >> gpurun_out/exp.txt 2>&1
HZG_POST_CHUNK=8192 python tools/sweep_time.py 16384 3 4 32 0 >> gpurun_out/exp.txt 2>&1
HZG_POST_CHUNK=16384 python tools/sweep_time.py 16384 3 4 32 0 >> gpurun_out/exp.txt 2>&1
HZG_POST_CHUNK=2048 python tools/sweep_time.py 16384 3 4 32 0 >> gpurun_out/exp.txt 2>&1
HZG_GROUPS=8 python tools/sweep_time.py 16384 3 4 32 0 >> gpurun_out/exp.txt 2>&1
HZG_GROUPS=32 python tools/sweep_time.py 16384 3 4 32 0 >> gpurun_out/exp.txt 2>&1
