#!/bin/bash
# Build a library variant ab/NAME.so: hv_tc.cu recompiled with extra nvcc
# defines (e.g. -DWGP_TC_ABLATE), every other object from the default build.
# usage: build_variant.sh NAME "DEFS" [hv_tc.cu-replacement]
set -e
cd "$(dirname "$0")/.."
name=$1; defs=$2; src=${3:-paper_2405_18328_b200/csrc/hv_tc.cu}
python -c "import paper_2405_18328_b200.build as b; b.build()" > /dev/null
mkdir -p ab/obj_$name
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -I include -I paper_2405_18328_b200/csrc -Xptxas -warn-spills"
$NV $FL $defs -c $src -o ab/obj_$name/hv_tc.o
objs=""
for o in paper_2405_18328_b200/_build/*.o; do
  [ "$(basename $o)" = hv_tc.o ] && objs="$objs ab/obj_$name/hv_tc.o" || objs="$objs $o"
done
$NV -gencode arch=compute_100a,code=sm_100a -shared -o ab/$name.so $objs -lcublas -lcusolver
echo ab/$name.so
