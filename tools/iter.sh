# build -> GPU tests -> bench (run under gpurun); one line summaries in gpurun_out/
mkdir -p gpurun_out
make -j8 > gpurun_out/i_build.log 2>&1 || { tail gpurun_out/i_build.log; exit 1; }
timeout 600 python -m pytest tests -x -q -m gpu ${TESTK:+-k "$TESTK"} > gpurun_out/i_gpu.log 2>&1; echo gpu_rc=$? >> gpurun_out/i_gpu.log
tail -2 gpurun_out/i_gpu.log
SVB_TRACE=1 timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err; echo bench_rc=$?
grep "jit pass" gpurun_out/i_bench.err | sort | uniq | head -8
python -c "import json;d=json.load(open('gpurun_out/i_bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],[round(p['ms'],3) for p in d['roofline']['passes']],d['dense']['ms_per_step'])"
