// fl_lib.cu -- single translation unit of libfftlattice_b200.so (the device
// twiddle table is a __device__ symbol shared by every kernel, so the kernels
// are compiled together instead of with relocatable device code).
#include "fl_sweep.cu"
#include "fl_conv.cu"
#include "fl_put.cu"
#include "fl_call.cu"
#include "fl_american.cu"
#include "fl_euro.cu"
#include "fl_fft.cu"
#include "fl_abi.cu"
#include "fl_dev.cu"
