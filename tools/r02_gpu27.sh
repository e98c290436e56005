mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svb_jit --launch-skip 6 --launch-count 1 -o gpurun_out/g27_syc_rb5 -f python tools/one_syc.py > gpurun_out/g27_ncu.log 2>&1; echo ncu_rc=$?; tail -2 gpurun_out/g27_ncu.log
