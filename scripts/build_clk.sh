# diagnostic build with per-phase clock64() counters (-DCT_PHASE_CLOCKS):
# paper_2102_05297_b200/libct_b200_clk.so, selected with CT_LIB_PATH
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -shared \
  -Xcompiler -fPIC -Xcompiler -ffp-contract=off -DCT_PHASE_CLOCKS -Iinclude \
  -Ipaper_2102_05297_b200/csrc paper_2102_05297_b200/csrc/ct_lib.cu \
  -o paper_2102_05297_b200/libct_b200_clk.so
