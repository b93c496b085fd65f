#!/bin/bash
# Measurement only: build variants/libdc_<name>.so = libdc.so with one source (default pc_owner.cu)
# compiled with extra flags (A/B of compile-time kernel shapes within one gpurun call; load with
# DC_SO_OVERRIDE).   [SRC=build.cu] bash tools/ab_variant.sh NAME -DFLAG=V ...
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
python -c "from paper_2411_02797_b200 import build; build.build()" > /dev/null
NI=$(python -c "import nvidia.nccl,os;print(list(nvidia.nccl.__path__)[0])")
mkdir -p variants
cd paper_2411_02797_b200
SRC=${SRC:-pc_owner.cu}
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -I ../include -I $NI/include \
  -DDC_HAVE_NCCL=1 "$@" -c csrc/$SRC -o /tmp/${SRC}_$NAME.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../variants/libdc_$NAME.so $(ls build_obj/*.o | grep -v $SRC) \
  /tmp/${SRC}_$NAME.o -L $NI/lib -l:libnccl.so.2 -Xlinker -rpath=$NI/lib
echo variants/libdc_$NAME.so
