# HBM optimizer kernels at C4 scale: default vs launch-shape variants; backward/forward ncu source
set -x
mkdir -p gpurun_out
for v in default w_mb2 w_ku1 w_ku3 r_kv1 r_kv3; do
  if [ $v = default ]; then L=""; else L="paper_2509_15645_b200/_build/var_$v/libgss_b200.so"; fi
  GSS_LIB=$L timeout 300 python tools/adam_probe.py 40000000 0.1292 >> gpurun_out/adam_probe_m.txt 2>&1
done
cat gpurun_out/adam_probe_m.txt | grep "{"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:backward_kernel -c 1 -o gpurun_out/c4_bwd_src python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_bwd.txt 2>&1
tail -2 gpurun_out/ncu_bwd.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:forward_kernel -s 9 -c 1 -o gpurun_out/c4_fwd_src python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_fwd.txt 2>&1
tail -2 gpurun_out/ncu_fwd.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"chain_kernel|slot_sum_kernel" -c 2 -o gpurun_out/c4_chain_src python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_chain.txt 2>&1
tail -2 gpurun_out/ncu_chain.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"duplicate_kernel|colour_kernel" -s 16 -c 2 -o gpurun_out/c4_dup_src python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_dup.txt 2>&1
tail -2 gpurun_out/ncu_dup.txt
