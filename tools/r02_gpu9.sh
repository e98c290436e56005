mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_dense.py tests/test_sharded_gloo.py tests/test_gpu_advice.py -q -m gpu -x > gpurun_out/g9_tests.log 2>&1; echo rc=$? >> gpurun_out/g9_tests.log; tail -5 gpurun_out/g9_tests.log
rm -rf /root/.cache/svb_jit
timeout 900 python tools/batch_probe.py > gpurun_out/g9_batch.json 2>&1; tail -2 gpurun_out/g9_batch.json
timeout 600 python tools/dense_bench.py 30 5 2>&1 | grep '"c64"\|"c128"' > gpurun_out/g9_dense.jsonl; grep fma gpurun_out/g9_dense.jsonl
