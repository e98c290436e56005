mkdir -p gpurun_out
for lib in build/bisect/5904446.so build/bisect/37189b1.so build/bisect/015aea3.so paper_2512_04216_b200/libsvb.so build/bisect/5904446.so; do
  SVB_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-configs --no-cpu-baseline > gpurun_out/g38_bench.json 2>gpurun_out/g38_bench.err
  echo "$lib $(python -c "import json;d=json.load(open('gpurun_out/g38_bench.json'));print(round(d['value']),round(d['ms_per_step'],3),round(d['roofline']['frac'],3),[round(p['ms'],3) for p in d['roofline']['passes']])")"
done
