// ops_kernels_3d.cu -- the 3D hexahedral (GLL) instantiations of the fused element
// operators and the BJ_ext block build (NEXT-4): advection and 3D Euler, N = 2, 3.
#define HBPDC_OPS_3D 1
#include "ops_kernels.cu"
