# build an A/B variant of libtwb200 with extra -D flags: scripts/build_variant.sh NAME FLAGS...
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -shared "$@" \
  -o paper_2601_00397_b200/lib/libtwb200_$name.so paper_2601_00397_b200/csrc/*.cu paper_2601_00397_b200/csrc/*.cpp
