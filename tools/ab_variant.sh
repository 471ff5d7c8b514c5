#!/bin/bash
# build ab/libmcinv_<name>.so: sweep6.cu recompiled with extra flags, linked with the
# current build_obj objects (compile-time A/B experiments; the product build is untouched)
# usage: tools/ab_variant.sh <name> <nvcc flags...>
set -e
cd "$(dirname "$0")/.."
name=$1; shift
O=paper_cs_0412107_b200/build_obj
src=${AB_SRC:-sweep6}
mkdir -p ab/obj_$name
for f in mcinv_host levels sweep sweep3 sweep5 sweep6 contract contract_ozaki reduce; do cp $O/$f.o ab/obj_$name/; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false -Xcompiler -fPIC,-O2 -cudart static -I include "$@" -c -o ab/obj_$name/$src.o paper_cs_0412107_b200/csrc/$src.cu
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ab/libmcinv_$name.so ab/obj_$name/*.o -lpthread
rm -rf ab/obj_$name
echo ab/libmcinv_$name.so
