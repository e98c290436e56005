mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass --launch-skip 6 --launch-count 1 -o gpurun_out/g36_interp -f python tools/one_batch_circ.py interp > gpurun_out/g36_ncu1.log 2>&1; tail -1 gpurun_out/g36_ncu1.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:svb_jit --launch-skip 6 --launch-count 1 -o gpurun_out/g36_jit -f python tools/one_batch_circ.py jit > gpurun_out/g36_ncu2.log 2>&1; tail -1 gpurun_out/g36_ncu2.log
