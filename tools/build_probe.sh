# probe build: lane-barrier wait cycles per phase in phase_cycles (see WB_PROBE in decode_kernel.cuh)
cd "$(dirname "$0")/../paper_1808_00687_b200/csrc" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static \
  -I../../include -DWB_PROBE -o ../_lib/libwfstb200_probe.so \
  wfst_decoder.cu lattice_host.cpp wfst_text.cpp posterior_io.cpp lattice_text.cpp
