# experiment builds: bash tools/build_variant.sh TAG [-DFLAG ...] -> _exp/libl1rxg_TAG.so
T=$1; shift
cd "$(dirname "$0")/.." && mkdir -p _exp
/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 -shared \
  -I include -I paper_1907_00463_b200/csrc "$@" -o _exp/libl1rxg_$T.so paper_1907_00463_b200/csrc/l1rxg.cu -lcudart -lcublas
