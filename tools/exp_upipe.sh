# one-round direct pass experiments (run under gpurun): ring depth, wait placement
mkdir -p gpurun_out
for cfg in "1 0" "1 1" "2 1" "2 0" "1 0"; do
  set -- $cfg
  SVB_UPIPE_AHEAD=$1 SVB_UWAIT_FIRST=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/x_$1_$2.json 2> gpurun_out/x_$1_$2.err
  echo "ahead=$1 waitfirst=$2 rc=$? $(python -c "import json;d=json.load(open('gpurun_out/x_$1_$2.json'));print(round(d['value']),round(d['ms_per_step'],3),round(d['roofline']['frac'],3),[round(p['ms'],3) for p in d['roofline']['passes']])" 2>&1 | tail -1)"
done
