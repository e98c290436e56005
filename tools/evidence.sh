# GPU evidence for profiles/: full -m gpu suite, smoke, bench (driver command), reference arm, ncu launch list
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/ev_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/ev_gpu_tests.log; tail -4 gpurun_out/ev_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/ev_smoke.log
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo bench_rc=$?; tail -3 gpurun_out/ev_bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; echo ref_rc=$?; cat gpurun_out/ev_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline > gpurun_out/ev_ncu_bench.log 2>&1; echo ncu_rc=$?
python -c "import json;d=json.load(open('gpurun_out/ev_bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d['cpu_baseline']['value'],d['clocks'])"
