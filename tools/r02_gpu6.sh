mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded_gloo.py -q -m gpu > gpurun_out/g6_sharded.log 2>&1; echo rc=$? >> gpurun_out/g6_sharded.log; tail -3 gpurun_out/g6_sharded.log
timeout 300 python bench.py --sharded --steps 5 --warmup 2 --no-cpu-baseline --no-configs > gpurun_out/g6_sharded_n1.json 2> gpurun_out/g6_sharded_n1.err; tail -2 gpurun_out/g6_sharded_n1.err; cat gpurun_out/g6_sharded_n1.json
rm -rf /root/.cache/svb_jit
SVB_BATCH_JIT_MIN_N=25 timeout 900 python tools/batch_probe.py > gpurun_out/g6_batch_nojit.json 2>&1; cat gpurun_out/g6_batch_nojit.json | tail -2
rm -rf /root/.cache/svb_jit
timeout 900 python tools/batch_probe.py > gpurun_out/g6_batch_jit.json 2>&1; cat gpurun_out/g6_batch_jit.json | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dense_tc --launch-count 1 -o gpurun_out/g6_dense_tc -f python tools/one_dense.py 5 > gpurun_out/g6_ncu_tc.log 2>&1; echo ncu_rc=$?
