// ops_kernels_gl_br2.cu -- the Navier-Stokes element operators with BR2 face gradients
// on Gauss-Legendre nodes (the paper's NS discretisation).
#define HBPDC_OPS_GL 1
#define HBPDC_OPS_BR2 1
#include "ops_kernels.cu"
