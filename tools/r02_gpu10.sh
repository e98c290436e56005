mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/g10_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/g10_gpu_tests.log; tail -4 gpurun_out/g10_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g10_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/g10_smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/g10_bench.json 2> gpurun_out/g10_bench.err; echo bench_rc=$?; tail -3 gpurun_out/g10_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/g10_ref.json 2> gpurun_out/g10_ref.err; echo ref_rc=$?; cat gpurun_out/g10_ref.json
python -c "import json;d=json.load(open('gpurun_out/g10_bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d['cpu_baseline']['value']);c=d['configs'];print(json.dumps({k:(v if k!='sycamore32_c64_1e6' else {kk:vv for kk,vv in v.items() if kk!='pass_table'}) for k,v in c.items()})[:4000])"
