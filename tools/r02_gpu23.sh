mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svb_jit --launch-skip 6 --launch-count 1 -o gpurun_out/g23_syc_ffma2 -f python tools/one_syc.py > gpurun_out/g23_ncu.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/g23_ncu.log
