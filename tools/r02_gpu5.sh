mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dense.py -q > gpurun_out/g5_dense.log 2>&1; echo rc=$? >> gpurun_out/g5_dense.log; tail -4 gpurun_out/g5_dense.log
timeout 900 python tools/batch_probe.py > gpurun_out/g5_batch_probe.json 2> gpurun_out/g5_batch_probe.err; cat gpurun_out/g5_batch_probe.json; tail -3 gpurun_out/g5_batch_probe.err
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err; echo bench_rc=$?; tail -5 gpurun_out/g5_bench.err
python -c "import json;d=json.load(open('gpurun_out/g5_bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['cpu_baseline']);print(json.dumps(d.get('configs'))[:3000])"
