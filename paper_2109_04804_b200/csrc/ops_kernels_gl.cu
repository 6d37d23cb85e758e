// ops_kernels_gl.cu -- the element operators and the BJ_ext block build on
// Gauss-Legendre nodes (NEXT-3): ops_kernels.cu instantiated with the
// GL face traces l_i(+-1) and surface weights lhat_i(+-1) (ops.cuh trace_load).
#define HBPDC_OPS_GL 1
#include "ops_kernels.cu"
