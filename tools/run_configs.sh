# bench + BASELINE configs 1, 3, 4 through the public API (run under gpurun)
set -x
python tools/configs.py ghz20 syc32 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
python tools/batch_bench.py --count 10000 > gpurun_out/batch.json 2> gpurun_out/batch.err
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ls -la gpurun_out
