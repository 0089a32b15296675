# sweep row-skip A/B; slot-sum ncu
set -x
mkdir -p gpurun_out
for v in default rskip rskip9 default; do
  if [ $v = default ]; then L=""; else L="paper_2509_15645_b200/_build/var_$v/libgss_b200.so"; fi
  echo "== $v" >> gpurun_out/time_render_r.txt
  GSS_LIB=$L timeout 300 python tools/time_render.py 40000000 3840 2160 >> gpurun_out/time_render_r.txt 2>&1
done
grep "==\|total" gpurun_out/time_render_r.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"slot_sum_depth_kernel" -s 1 -c 1 -o gpurun_out/c4_ssum_src python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_ssum.txt 2>&1
tail -1 gpurun_out/ncu_ssum.txt
