# round-2 first GPU pass: host facts + link probe, C4 bench probes, full -m gpu suite, scale parity
set -x
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20; nvidia-smi topo -m; nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" | head -20) > gpurun_out/host.txt 2>&1
timeout 120 tools/linkprobe > gpurun_out/linkprobe.txt 2>&1
timeout 600 python bench.py --gaussians 40000000 --width 3840 --height 2160 --steps 5 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/c4_hbm.json 2> gpurun_out/c4_hbm.err
timeout 600 python bench.py --gaussians 18000000 --steps 5 --warmup 3 --no-cpu-baseline --no-probe --nongeo-on-host > gpurun_out/c3_host.json 2> gpurun_out/c3_host.err
export GSS_PARITY_OUT=$PWD/gpurun_out/parity.json
timeout 1200 python -m pytest tests -x -q -m gpu --ignore=tests/test_scale_parity_gpu.py > gpurun_out/pytest_gpu.txt 2>&1
timeout 2400 python -m pytest tests/test_scale_parity_gpu.py -q -m gpu --durations=10 > gpurun_out/pytest_scale.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt gpurun_out/pytest_scale.txt
