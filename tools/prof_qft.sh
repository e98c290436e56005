# ncu evidence for the QFT-30 bench (run under gpurun; outputs in gpurun_out/)
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
# the dominant kernel of the bench step: the last fused pass (zero-start, fused <Z>)
ncu --set full --import-source on --clock-control none -k regex:svb_jit --launch-skip 3 --launch-count 1 -o gpurun_out/qft30_top -f python tools/one_apply.py 30 c128 z > gpurun_out/ncu_full.log 2>&1
# a full-stream pass of the dense-input program (second apply: pass 1)
ncu --set full --import-source on --clock-control none -k regex:svb_jit --launch-skip 5 --launch-count 1 -o gpurun_out/qft30_dense -f python tools/one_apply.py 30 c128 z2 > gpurun_out/ncu_dense.log 2>&1
ls -la gpurun_out
