mkdir -p gpurun_out
timeout 900 python tools/batch_pass_probe.py > gpurun_out/g28_passes.txt 2>&1; cat gpurun_out/g28_passes.txt | cut -c1-600
