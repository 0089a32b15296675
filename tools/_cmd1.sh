set -x
nproc; free -g; lscpu | head -20; nvidia-smi topo -m; nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" | head -20
timeout 120 tools/linkprobe > gpurun_out/linkprobe.txt 2>&1; cat gpurun_out/linkprobe.txt
timeout 600 python bench.py --gaussians 40000000 --width 3840 --height 2160 --steps 5 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/c4_hbm.json 2> gpurun_out/c4_hbm.err; tail -c 3000 gpurun_out/c4_hbm.json; tail -20 gpurun_out/c4_hbm.err
timeout 600 python bench.py --gaussians 40000000 --width 3840 --height 2160 --steps 3 --warmup 3 --no-cpu-baseline --no-probe --nongeo-on-host > gpurun_out/c4_host.json 2> gpurun_out/c4_host.err; tail -c 3000 gpurun_out/c4_host.json; tail -20 gpurun_out/c4_host.err
