mkdir -p gpurun_out
timeout 300 ./tools/mb/d2hbench > gpurun_out/g42_d2h.txt 2>&1; cat gpurun_out/g42_d2h.txt
nvidia-smi -q | grep -i "Link Width\|Link Gen\|Current\s*:\|Max\s*:" | head -12
