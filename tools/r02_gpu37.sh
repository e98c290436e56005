mkdir -p gpurun_out
SVB_JIT_STRICT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "initial_permutation or permuted or zero_start or fused_z" > gpurun_out/g37_tests.log 2>&1; tail -3 gpurun_out/g37_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-configs --no-cpu-baseline > gpurun_out/g37_bench.json 2>gpurun_out/g37_bench.err; python -c "import json;d=json.load(open('gpurun_out/g37_bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['dense']['ms_per_step'],[round(p['ms'],2) for p in d['dense']['passes']])"
