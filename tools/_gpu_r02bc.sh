# ncu --set full of the final sweep (folded exp factor) at C4 camera 0
set -x
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:backward_kernel -c 1 -o gpurun_out/c4_bwd_bc python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_bwd_bc.txt 2>&1
tail -n 1 gpurun_out/ncu_bwd_bc.txt
