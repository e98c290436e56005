mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dense.py tests/test_gpu_batch.py tests/test_gpu_parity.py -q -x > gpurun_out/g18_tests.log 2>&1; echo rc=$? >> gpurun_out/g18_tests.log; tail -4 gpurun_out/g18_tests.log
timeout 1200 python tools/batch_probe.py > gpurun_out/g18_batch.json 2> gpurun_out/g18_batch.err; cat gpurun_out/g18_batch.json; tail -3 gpurun_out/g18_batch.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-configs --no-cpu-baseline > gpurun_out/g18_bench.json 2>gpurun_out/g18_bench.err; python -c "import json;d=json.load(open('gpurun_out/g18_bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['dense']['ms_per_step'])"
