# Builds an A/B variant of the engine library: tools/build_ab.sh NAME "-DFOO=1 ..."
# -> tools/ab_NAME.so (select it at run time with MHAR_LIB=tools/ab_NAME.so)
set -e
cd "$(dirname "$0")/../paper_2104_07097_b200/csrc"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr $2 -shared \
  -o ../../tools/ab_$1.so abi.cu group.cu host_linalg.cpp lp.cu -lcudart -ldl
