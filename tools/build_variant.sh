# build a variant library: tools/build_variant.sh NAME -DFLAG ... -> _lib/libwfstb200_NAME.so
name=$1; shift
cd "$(dirname "$0")/../paper_1808_00687_b200/csrc" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static \
  -I../../include "$@" -o ../_lib/libwfstb200_$name.so \
  wfst_decoder.cu lattice_host.cpp wfst_text.cpp posterior_io.cpp lattice_text.cpp
