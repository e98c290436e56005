# in-body uniform-slot wait (UIN) vs the loop's wait, same box (run under gpurun)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/u_gpu.log 2>&1; echo gpu_rc=$? >> gpurun_out/u_gpu.log; tail -2 gpurun_out/u_gpu.log
for v in 1 0 1 0; do
  SVB_UIN=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/u_$v.json 2> gpurun_out/u_$v.err
  echo "uin=$v rc=$? $(python -c "import json;d=json.load(open('gpurun_out/u_$v.json'));print(round(d['value']),round(d['ms_per_step'],3),round(d['roofline']['frac'],3),[round(p['ms'],3) for p in d['roofline']['passes']])" 2>&1 | tail -1)"
done
