mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-configs --no-cpu-baseline > gpurun_out/g39_bench.json 2>gpurun_out/g39_bench.err
python -c "import json;d=json.load(open('gpurun_out/g39_bench.json'));print(round(d['value']),round(d['ms_per_step'],3),round(d['roofline']['frac'],3),[round(p['ms'],3) for p in d['roofline']['passes']], d['dense']['ms_per_step'])"
SVB_JIT_STRICT=1 timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/g39_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/g39_gpu_tests.log; tail -3 gpurun_out/g39_gpu_tests.log
