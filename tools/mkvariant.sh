#!/bin/bash
# tooling: build paper_2411_14315_b200/variants/libhbgpu_$TAG.so from the objects of the
# default build, recompiling only the listed sources with extra -D flags
#   tools/mkvariant.sh TAG "-DTAN_G2=4" hbgpu_tangent_pipe.cu [more.cu]
set -e
TAG=$1; DEFS=$2; shift 2
cd "$(dirname "$0")/../paper_2411_14315_b200/csrc"
mkdir -p ../variants ../_obj_$TAG
OBJS=""
for f in hbgpu_kernels hbgpu_tangent hbgpu_tangent_pipe hbgpu_matvec hbgpu_krylov hbgpu_time hbgpu_host; do
  if [[ " $* " == *" $f.cu "* ]]; then
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I../../include $DEFS -c $f.cu -o ../_obj_$TAG/$f.o
    OBJS="$OBJS ../_obj_$TAG/$f.o"
  else
    OBJS="$OBJS ../_obj/$f.o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../variants/libhbgpu_$TAG.so $OBJS
echo built $TAG
