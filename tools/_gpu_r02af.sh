# ncu of the deferred update passes at C4 scale (steady-state counters)
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"walk4_kernel|update_kernel|restore_walk" -s 60 -c 3 -o gpurun_out/adam_c4 python tools/adam_probe.py 40000000 0.1292 > gpurun_out/ncu_adam.txt 2>&1
tail -n 2 gpurun_out/ncu_adam.txt
