set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/b.json 2> gpurun_out/b.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:svb_jit --launch-skip 1 --launch-count 1 -o gpurun_out/qft30_pass1 -f python tools/one_apply.py 30 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
