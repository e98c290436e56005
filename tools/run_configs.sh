# bench + BASELINE configs 1, 3, 4 through the public API (run under gpurun)
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python tools/configs.py ghz20 syc32 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
python tools/batch_bench.py --count 10000 > gpurun_out/batch.json 2> gpurun_out/batch.err
python tools/batch_bench.py --count 10000 --workers 8 >> gpurun_out/batch.json 2>> gpurun_out/batch.err
timeout 300 python bench.py --sharded --steps 3 --warmup 1 > gpurun_out/sharded1.json 2> gpurun_out/sharded1.err
ls -la gpurun_out
