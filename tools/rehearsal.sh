# what the driver runs at round end, in order (run under gpurun)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r_build.log 2>&1; echo build_rc=$? >> gpurun_out/r_build.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/r_smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r_gpu.log 2>&1; echo gpu_rc=$? >> gpurun_out/r_gpu.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r_ref.json 2> gpurun_out/r_ref.err; echo ref_rc=$? >> gpurun_out/r_ref.err
timeout 900 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo bench_rc=$? >> gpurun_out/r_bench.err
