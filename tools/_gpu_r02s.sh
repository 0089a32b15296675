# composite launch-shape variants (pixels per thread, batch, blocks/SM)
set -x
mkdir -p gpurun_out
for v in default fppt4 fb128 fminb3 default; do
  if [ $v = default ]; then L=""; else L="paper_2509_15645_b200/_build/var_$v/libgss_b200.so"; fi
  echo "== $v" >> gpurun_out/time_render_s.txt
  GSS_LIB=$L timeout 300 python tools/time_render.py 40000000 3840 2160 >> gpurun_out/time_render_s.txt 2>&1
done
grep "==\|total" gpurun_out/time_render_s.txt
