# build tuning variants of libsieve.so: tools/build_variants.sh NAME "-DFLAG=.." ...
set -e
NAME=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  paper_1205_4883_b200/csrc/kernels.cu paper_1205_4883_b200/csrc/primality.cu paper_1205_4883_b200/csrc/peer.cu paper_1205_4883_b200/csrc/runtime.cu -o build/libsieve_$NAME.so
