# developer: build a variant of the library with extra nvcc defines into variants/libevoke_NAME.so
#   bash tools/build_variant.sh NAME -DFOO=1 ...   (A/B with EVOKE_LIB_PATH=variants/libevoke_NAME.so)
set -e
name=$1; shift
mkdir -p variants
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  -diag-suppress 177,550 "$@" -o variants/libevoke_$name.so paper_1911_10616_b200/csrc/evoke.cu
