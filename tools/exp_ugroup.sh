# tiles per uniform slot (SVB_UGROUP) on the one-round direct pass, same box (run under gpurun)
mkdir -p gpurun_out
SVB_UGROUP=2 SVB_JIT_STRICT=1 timeout 600 python -m pytest tests -x -q -m gpu -k "qft or zsum or jit or smoke" 2>&1 | tail -1
for v in 1 2 4 1 2 4; do
  SVB_UGROUP=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/g_$v.json 2> gpurun_out/g_$v.err
  echo "group=$v rc=$? $(python -c "import json;d=json.load(open('gpurun_out/g_$v.json'));print(round(d['value']),round(d['ms_per_step'],3),round(d['roofline']['frac'],3),[round(p['ms'],3) for p in d['roofline']['passes']])" 2>&1 | tail -1)"
done
