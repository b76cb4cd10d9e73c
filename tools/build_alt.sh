#!/bin/bash
# A/B builds: libb2moe_alt.so = the library with extra nvcc defines (e.g. -DB2_DGRAD_STAGED_GU),
# loaded by setting B2_LIB=paper_2604_00785_b200/libb2moe_alt.so. Usage: bash tools/build_alt.sh -DNAME ...
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
python -c "import sys; sys.path.insert(0, '$ROOT'); from paper_2604_00785_b200 import _build; _build.build()"
mkdir -p $ROOT/build/obj_alt
NVCC=/usr/local/cuda/bin/nvcc
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I $ROOT/paper_2604_00785_b200/csrc -I $ROOT/include"
OBJS=""
for f in $ROOT/paper_2604_00785_b200/csrc/*.cu $ROOT/paper_2604_00785_b200/csrc/*.cpp; do
  b=$(basename $f)
  if grep -q "B2_DGRAD_STAGED_GU\|B2_ALT" $f; then
    $NVCC $FLAGS "$@" -c $f -o $ROOT/build/obj_alt/$b.o; OBJS="$OBJS $ROOT/build/obj_alt/$b.o"
  else
    OBJS="$OBJS $ROOT/build/obj/$b.o"
  fi
done
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/paper_2604_00785_b200/libb2moe_alt.so $OBJS -lnccl
echo built $ROOT/paper_2604_00785_b200/libb2moe_alt.so
