mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_resident.py -q > gpurun_out/g7_tests.log 2>&1; echo rc=$? >> gpurun_out/g7_tests.log; tail -25 gpurun_out/g7_tests.log
cat gpurun_out/resident_calls.json; echo
timeout 600 python tools/dense_bench.py 30 5 > gpurun_out/g7_dense_bench.jsonl 2> gpurun_out/g7_dense_bench.err; cat gpurun_out/g7_dense_bench.jsonl | grep '"c64"'; tail -3 gpurun_out/g7_dense_bench.err
rm -rf /root/.cache/svb_jit
timeout 900 python tools/batch_probe.py > gpurun_out/g7_batch_jit.json 2>&1; tail -2 gpurun_out/g7_batch_jit.json
timeout 300 python bench.py --sharded --steps 5 --warmup 2 --no-cpu-baseline --no-configs > gpurun_out/g7_sharded_n1.json 2> gpurun_out/g7_sharded_n1.err; tail -2 gpurun_out/g7_sharded_n1.err; python -c "import json;d=json.load(open('gpurun_out/g7_sharded_n1.json'));print(d['value'],d['ms_per_step'])"
