#!/bin/bash
# Build libbhrt_b200 variants differing only in -D macros into build/variants/
# (developer tuning; time them with BHRT_B200_LIB=... python tools/quick_time.py).
#   spec = name:-DFOO=1,-DBAR=2        sources from the working tree
#   spec = name@REF:-DFOO=1            sources from git revision REF
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -std=c++17 -lineinfo --fmad=false -Xcompiler -fPIC,-ffp-contract=off -Iinclude"
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}; defs=${defs//,/ }
  src=paper_2507_16165_b200/csrc
  inc=include
  if [[ "$name" == *@* ]]; then
    ref=${name#*@}; name=${name%%@*}
    root=build/variants/src_$name
    rm -rf "$root"; mkdir -p "$root"
    git archive "$ref" paper_2507_16165_b200/csrc include | tar -x -C "$root"
    src=$root/paper_2507_16165_b200/csrc
    inc=$root/include
  fi
  objs=""
  for f in trace_reference.cu trace_scene.cu table.cu shade.cu bhrt_cuda.cu fp64_peak.cu scene_text.cpp; do
    nvcc $ARCH ${FL/-Iinclude/-I$inc} -I$src $defs -c $src/$f -o build/variants/${name}_${f%.*}.o &
    objs="$objs build/variants/${name}_${f%.*}.o"
  done
  wait
  nvcc $ARCH -shared -o build/variants/lib_$name.so $objs -lcudart
  rm -f $objs
  [[ "$src" == build/variants/src_* ]] && rm -rf "build/variants/src_$name"
  echo built build/variants/lib_$name.so
done
