# bench + BASELINE configs 1, 3, 4 through the public API + ncu evidence (run under gpurun)
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python tools/qft_probe.py > gpurun_out/probe.jsonl 2>&1
python tools/configs.py ghz20 syc32 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
python tools/batch_bench.py --count 10000 > gpurun_out/batch.json 2> gpurun_out/batch.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:svb_jit --launch-skip 3 --launch-count 1 -o gpurun_out/qft30_top -f python tools/one_apply.py 30 c128 z > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:svb_jit --launch-skip 5 --launch-count 1 -o gpurun_out/qft30_dense -f python tools/one_apply.py 30 c128 z2 > gpurun_out/ncu_dense.log 2>&1
ls -la gpurun_out
