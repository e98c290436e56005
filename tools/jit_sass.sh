#!/bin/bash
# Dump the JIT sources of a QFT-n (or other suite) program and count SASS per pass (CPU only).
# usage: tools/jit_sass.sh [n] [prec 0|1]
n=${1:-30}; prec=${2:-1}
cd "$(dirname "$0")/.."
rm -f /tmp/jit_pass*.cu
SVB_JIT_DUMP=/tmp/jit_all.cu python - "$n" "$prec" <<'PY'
import ctypes, sys
from paper_2512_04216_b200 import _lib, suite, statevector as sv
n, prec = int(sys.argv[1]), int(sys.argv[2], 0)
import os
c = suite.sycamore_circuit(4, 8, 20, 0, measured=False) if os.environ.get("SYC") else suite.qft_bench_circuit(n)
g = sv.gate_array(c.instructions)
cb = ctypes.c_int64(); buf = ctypes.create_string_buffer(4096)
rc = _lib.lib().svb_jit_check(n, prec, g.ctypes.data_as(ctypes.c_void_p), g.size, ctypes.byref(cb), buf, 4096)
assert rc == 0, buf.value
s = open('/tmp/jit_all.cu').read()
parts = s.split('#include "device_core.cuh"')[1:]
for k, p in enumerate(parts):
    open(f'/tmp/jit_pass{k}.cu', 'w').write('#include "device_core.cuh"' + p)
PY
for f in /tmp/jit_pass*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -cubin -O3 -Ipaper_2512_04216_b200/csrc -std=c++17 -o ${f%.cu}.cubin $f -Xptxas -v 2>&1 | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores" | tr '\n' ' '
  cuobjdump -sass ${f%.cu}.cubin | grep -oE "^\s+/\*[0-9a-f]+\*/\s+[A-Z0-9.]+" | awk '{print $2}' | sed 's/\..*//' | sort | uniq -c | sort -rn | awk '$2 ~ /^(DFMA|DMUL|DADD|LDS|STS|IMAD|SHFL)$/' | tr -s ' \n' ' '
  echo
done
