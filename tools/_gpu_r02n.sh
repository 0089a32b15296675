# sweep software-pipelined reduction A/B; optimizer launch-shape variants; chain/dup/colour ncu
set -x
mkdir -p gpurun_out
for v in default bp10 bp9 bp8 default; do
  if [ $v = default ]; then L=""; else L="paper_2509_15645_b200/_build/var_$v/libgss_b200.so"; fi
  echo "== $v" >> gpurun_out/time_render_n.txt
  GSS_LIB=$L timeout 300 python tools/time_render.py 40000000 3840 2160 >> gpurun_out/time_render_n.txt 2>&1
done
grep "==\|total" gpurun_out/time_render_n.txt
GSS_LIB=paper_2509_15645_b200/_build/var_bp10/libgss_b200.so timeout 600 python -m pytest tests/test_raster_gpu.py -x -q > gpurun_out/pytest_n_bp10.txt 2>&1; tail -2 gpurun_out/pytest_n_bp10.txt
for v in default w_ku1 w1_mb5 w1_mb6 w1_mb4_g16 r_kv1 r1_mb6 r1_mb8; do
  if [ $v = default ]; then L=""; else L="paper_2509_15645_b200/_build/var_$v/libgss_b200.so"; fi
  GSS_LIB=$L timeout 300 python tools/adam_probe.py 40000000 0.1292 >> gpurun_out/adam_probe_n.txt 2>&1
done
grep "{" gpurun_out/adam_probe_n.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"chain_kernel|slot_sum_kernel" -c 2 -o gpurun_out/c4_chain_src python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_chain.txt 2>&1
tail -1 gpurun_out/ncu_chain.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"duplicate_kernel|colour_kernel" -s 16 -c 2 -o gpurun_out/c4_dup_src python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_dup.txt 2>&1
tail -1 gpurun_out/ncu_dup.txt
