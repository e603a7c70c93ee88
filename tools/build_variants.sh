#!/bin/bash
# Build libbhrt_b200 variants differing only in -D macros into build/variants/
# (developer tuning; time them with BHRT_B200_LIB=... python tools/quick_time.py).
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -std=c++17 -lineinfo --fmad=false -Xcompiler -fPIC,-ffp-contract=off -Iinclude"
for spec in "$@"; do   # spec: name:-DFOO=1,-DBAR=2
  name=${spec%%:*}; defs=${spec#*:}; defs=${defs//,/ }
  objs=""
  for f in trace_reference trace_scene table shade bhrt_cuda fp64_peak; do
    nvcc $ARCH $FL $defs -c paper_2507_16165_b200/csrc/$f.cu -o build/variants/${name}_$f.o
    objs="$objs build/variants/${name}_$f.o"
  done
  nvcc $ARCH -shared -o build/variants/lib_$name.so $objs -lcudart
  echo built build/variants/lib_$name.so
done
